"""N>1 host path on CPU: world_size-2 gloo processes shard the hypotheses,
score their shard (CPU oracle stands in for the GPU kernel here), all-gather,
and reduce; every rank must end with the single-process result, bitwise."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    from helpers import cfg1_oracle
    from oracle import pyoracle as O
    from paper_2312_08715_b200.shard import gather_scores, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = cfg1_oracle()
    poses = w.grid_poses()[:203]  # uneven shards
    lo, hi = shard_range(poses.shape[0], rank, world)
    s, _ = O.score_poses(w.k, w.observed, w.vertices, w.triangles, poses[lo:hi], w.noise,
                         w.sigma_max, w.window, threads=2)
    allv = gather_scores(torch.from_numpy(s), poses.shape[0], world).numpy()
    probs, _ = O.normalize(allv[:, 0])
    res = np.array([O.argmax(allv[:, 0]), O.sample_categorical(probs, O.rng_seed(7)),
                    O.logsumexp(allv[:, 0])])
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.concatenate([allv[:, 0], res]))
    dist.destroy_process_group()


def test_two_rank_gloo_shard_gather_reduce(tmp_path, oracle):
    import torch.multiprocessing as mp
    from helpers import cfg1_oracle
    port = 29500 + (os.getpid() % 1000)
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "r0.npy")
    r1 = np.load(tmp_path / "r1.npy")
    assert np.array_equal(r0, r1)
    w = cfg1_oracle()
    poses = w.grid_poses()[:203]
    s, _ = oracle.score_poses(w.k, w.observed, w.vertices, w.triangles, poses, w.noise,
                              w.sigma_max, w.window, threads=2)
    assert np.array_equal(r0[:203], s[:, 0])
    probs, _ = oracle.normalize(s[:, 0])
    assert r0[203] == oracle.argmax(s[:, 0])
    assert r0[204] == oracle.sample_categorical(probs, oracle.rng_seed(7))


def test_shard_range_partitions():
    sys.path.insert(0, ROOT)
    from paper_2312_08715_b200.shard import shard_range
    for n in (0, 1, 7, 1024, 1048576):
        for world in (1, 2, 3, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
