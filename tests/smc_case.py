"""A small scene-graph inference case shared by the SMC tests (oracle on CPU,
device SMC on the GPU): a 0.3 x 0.3 m table seen from 0.5 m above, a
two-object library of seeded voxel blobs, one (or two) placed objects in the
observation."""
import numpy as np

from paper_2312_08715_b200 import configs, synth

K = configs.Intr(70.0, 70.0, 24.0, 18.0, 48, 36, 0.01, 5.0)
CAMERA = np.array([0.0, 1.0, 0.0, 0.0, 0.0, 0.0, 0.5])  # looking straight down
TABLE_W = TABLE_H = 0.3
NOISE_GRID = [(p, f * 0.1) for p in (0.05, 0.3, 0.8) for f in (0.25, 0.5, 1.0)]
SCHEDULE = ((3, 3, 4), [(2, 2, 2)])


def build(mesh_fn, box_fn, contact_fn, render_scene, n_placed=1):
    lib = []
    for i, n in enumerate((150, 260)):
        v, t = configs.make_mesh(synth.eden_blob(n, 40 + i), mesh_fn)
        lib.append((v, t, v.min(axis=0), v.max(axis=0)))
    tv, tt, _, _ = configs.table_mesh(box_fn, TABLE_W, TABLE_H)
    placed = [(1, 1, 0.08, 0.11, 1.3), (0, 2, 0.17, 0.05, 4.0)][:n_placed]
    inst = [(tv, tt, np.array([1.0, 0, 0, 0, 0, 0, 0]))]
    for obj, face, dx, dy, dt in placed:
        pose = contact_fn(TABLE_W, TABLE_H, lib[obj][2], lib[obj][3], face, dx, dy, dt)
        inst.append((lib[obj][0], lib[obj][1], pose))
    depth = render_scene(K, CAMERA, inst)
    rng = np.random.Generator(np.random.PCG64(77))
    obs = synth.noisy_observation(depth, K.far, 0.002, 0.03, 0.2, 1.0, rng, K.near)
    return lib, (tv, tt), obs, placed
