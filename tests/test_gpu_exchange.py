"""GPU: the sharded stage exchange on one rank.

Only one GPU is available to the build, so the multi-rank behaviour is
covered by construction plus these single-rank checks of the same code: the
peer stores honour their capacity and only the score-many paths use them;
b3d_gpu_enumerate_shard alternates the halves of the global array per epoch
(two consecutive steps with different scores: neither overwrites the other's
half, each result equals the plain single-call enumeration); the signal-pad
barrier and the symmetric-memory allocation through a 1-rank NCCL group.
"""
import numpy as np
import pytest
import torch

from helpers import b3d_intr, cfg1_oracle
from paper_2312_08715_b200 import b3d

pytestmark = pytest.mark.gpu


def _setup(ctx):
    w = cfg1_oracle()
    ctx.set_camera(b3d_intr(w.k))
    mid = ctx.upload_mesh(w.vertices, w.triangles)
    ctx.set_observation(w.observed)
    ctx.set_likelihood(w.noise, w.sigma_max, w.window)
    return w, mid


def test_peer_stores_respect_capacity_and_paths(gpu_ctx):
    w, mid = _setup(gpu_ctx)
    poses = w.grid_poses()[:200]
    peer = torch.full((200,), -7.0, dtype=torch.float64, device="cuda")
    sc = torch.zeros((200, 1), dtype=torch.float64, device="cuda")
    gpu_ctx.set_score_peers([peer.data_ptr()], 50, 120)  # rows 50.. but only elements < 120
    try:
        gpu_ctx.score_poses(mid, torch.from_numpy(poses).cuda(), sc, None)
        torch.cuda.synchronize()
        assert (peer[:50] == -7).all() and (peer[120:] == -7).all()
        assert torch.equal(peer[50:120], sc[:70, 0])
        # camera-mode / contact / chain paths never store to peers
        peer.fill_(-7.0)
        o = w.vertices
        g = b3d.ContactGrid.make(0.5, 0.5, o.min(axis=0), o.max(axis=0), 1, (2, 2, 2))
        gpu_ctx.score_contact_grid(mid, g)
        gpu_ctx.coarse_to_fine(mid, w.gt_pose, [{"extent": w.extent, "count": (2, 2, 2),
                                                 "rotations": w.rotations[:2], "mode": 0,
                                                 "noise": w.noise[0], "window": 1, "select": 1}])
        torch.cuda.synchronize()
        assert (peer == -7).all()
    finally:
        gpu_ctx.set_score_peers([], 0)
    # chunked settings (> 12 entries) still deliver every column to the peer
    noise = [(0.01 * (i + 1), 0.005) for i in range(14)]
    gpu_ctx.set_likelihood(noise, 0.1, 1)
    big = torch.full((14 * 200,), -7.0, dtype=torch.float64, device="cuda")
    sc14 = torch.zeros((200, 14), dtype=torch.float64, device="cuda")
    gpu_ctx.set_score_peers([big.data_ptr()], 0, 14 * 200)
    try:
        gpu_ctx.score_poses(mid, torch.from_numpy(poses).cuda(), sc14, None)
        torch.cuda.synchronize()
        assert torch.equal(big.view(200, 14), sc14)
    finally:
        gpu_ctx.set_score_peers([], 0)
        gpu_ctx.set_likelihood(w.noise, w.sigma_max, w.window)


def test_enumerate_shard_alternates_halves(gpu_ctx):
    """Two consecutive exchanges with different observations: exchange e
    writes half (e & 1) only, so step 2 never touches what step 1's reducer
    reads; each result equals enumerate_poses on that step's inputs."""
    w, mid = _setup(gpu_ctx)
    n = 256
    poses = w.grid_poses()[:n]
    obs2 = w.observed.copy()
    obs2[40:80, 60:100] = 0.45  # a different frame: different scores
    arr = torch.full((2 * n, 1), np.nan, dtype=torch.float64, device="cuda")
    sig = torch.zeros(1, dtype=torch.int64, device="cuda")
    outs, halves = [], []
    for epoch, obs in ((1, w.observed), (2, obs2)):
        ex = b3d.ShardExchange.make(0, 0, n, [arr.data_ptr()], [sig.data_ptr()], epoch)
        st = b3d.rng_seed(3)
        outs.append((gpu_ctx.enumerate_shard(mid, ex, poses=poses, depth=obs, rng_state=st), st))
        torch.cuda.synchronize()
        halves.append(arr.clone())
    h1, h2 = halves
    assert torch.isnan(h1[:n]).all() and torch.equal(h2[n:], h1[n:])  # epoch 1 -> half 1
    assert not torch.isnan(h2[:n]).any() and not torch.equal(h2[:n], h2[n:])
    assert int(sig[0].item()) == 2
    for (res, st), obs, half in zip(outs, (w.observed, obs2), (h1[n:], h2[:n])):
        st_ref = b3d.rng_seed(3)
        sc = np.zeros((n, 1))
        ref = gpu_ctx.enumerate_observed(mid, obs, poses, rng_state=st_ref, scores=sc)
        np.testing.assert_array_equal(half.cpu().numpy(), sc)
        assert (res.argmax, res.sample, res.max_score, res.logsumexp) == \
            (ref.argmax, ref.sample, ref.max_score, ref.logsumexp)
        np.testing.assert_array_equal(st, st_ref)


def test_enumerate_shard_on_symmetric_memory_single_rank(gpu_ctx):
    """SymmetricExchange (torch symmetric memory through a 1-rank NCCL group)
    + the device pose grid path, against enumerate_grid."""
    import socket
    import torch.distributed as dist
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
    except Exception:
        pytest.skip("symmetric memory unavailable")
    from paper_2312_08715_b200.shard import SymmetricExchange
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        w, mid = _setup(gpu_ctx)
        d_rot = torch.from_numpy(w.rotations).cuda()
        grid = gpu_ctx.make_grid(w.center, w.extent, w.count, d_rot, w.grid_mode)
        n = w.n_hyp
        try:
            xch = SymmetricExchange(n, 1, torch.device("cuda", 0))
        except Exception as e:
            pytest.skip(f"symmetric memory rendezvous unavailable: {e}")
        d_res = torch.zeros(64, dtype=torch.uint8, device="cuda")
        d_rng = torch.from_numpy(b3d.rng_seed(7).view(np.int64)).cuda()
        ref_res = torch.zeros(64, dtype=torch.uint8, device="cuda")
        ref_rng = d_rng.clone()
        ref_sc = torch.zeros((n, 1), dtype=torch.float64, device="cuda")
        for _ in range(3):
            gpu_ctx.enumerate_shard(mid, xch.exchange(0), grid=grid, n_local=n, rng_state=d_rng,
                                    out=d_res)
            gpu_ctx.enumerate_grid(mid, grid, ref_rng, ref_res, ref_sc)
            torch.cuda.synchronize()
            assert torch.equal(xch.half(), ref_sc)
            assert torch.equal(d_res, ref_res) and torch.equal(d_rng, ref_rng)
    finally:
        dist.destroy_process_group()


def test_enumerate_observed_graph_replay_tracks_inputs(gpu_ctx):
    """b3d_gpu_enumerate_observed with page-locked buffers is captured into a
    CUDA graph on its second call and replayed afterwards: the replays read
    the buffers' current contents (new observation / poses / Rng state every
    call) and equal the plain path exactly; a setter invalidates the graph."""
    w, mid = _setup(gpu_ctx)
    n = 512
    h_obs = torch.from_numpy(w.observed).pin_memory().numpy()
    h_poses = torch.from_numpy(w.grid_poses()[:n]).pin_memory().numpy()
    h_sc = torch.zeros((n, 1), dtype=torch.float64).pin_memory().numpy()
    rng = np.random.Generator(np.random.PCG64(4))
    for it in range(6):
        obs = w.observed.copy()
        y, x = rng.integers(0, 100), rng.integers(0, 140)
        obs[y:y + 20, x:x + 20] = np.float32(0.3 + 0.05 * it)
        h_obs[:] = obs
        h_poses[:] = w.grid_poses()[it * 64:it * 64 + n]
        st = b3d.rng_seed(100 + it)
        res = gpu_ctx.enumerate_observed(mid, h_obs, h_poses, rng_state=st, scores=h_sc)
        # plain reference: device buffers, separate calls
        gpu_ctx.set_observation(torch.from_numpy(obs).cuda())
        ref_sc, _ = gpu_ctx.score_poses(mid, w.grid_poses()[it * 64:it * 64 + n])
        st_ref = b3d.rng_seed(100 + it)
        ref = gpu_ctx.stage_reduce(ref_sc[:, 0], rng_state=st_ref)
        np.testing.assert_array_equal(h_sc, ref_sc)
        assert (res.argmax, res.sample, res.max_score, res.logsumexp) == \
            (ref.argmax, ref.sample, ref.max_score, ref.logsumexp)
        np.testing.assert_array_equal(st, st_ref)
        if it == 3:  # a setter in between: the next call recaptures
            gpu_ctx.set_likelihood([(0.02, 0.006)], w.sigma_max, 2)
    gpu_ctx.set_likelihood(w.noise, w.sigma_max, w.window)


@pytest.mark.gpu
@pytest.mark.parametrize("n_ranks", [2, 3, 4, 8])
def test_exchange_protocol_emulated_ranks(gpu_ctx, n_ranks):
    """The exchange protocol for 2-8 ranks, every rank one block of one
    cooperative launch on this GPU (the recipe's stand-in for more GPUs):
    stores into every rank's array half, signal-pad barrier with growing
    epochs, own-half reads with one slow reader per epoch.  Double-buffered
    (the product's layout): no reader ever sees a peer's next-epoch value.
    Single-buffered (control): the slow reader does -- the race the halves
    remove, so the test can see it."""
    assert gpu_ctx.exchange_emulation(n_ranks, 200, double_buffered=True, hold_ns=20_000) == 0
    assert gpu_ctx.exchange_emulation(n_ranks, 50, double_buffered=False, hold_ns=50_000) > 0
