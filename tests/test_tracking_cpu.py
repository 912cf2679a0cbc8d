"""Camera tracking (track_camera, tracking.cpp:59-172) host pieces on CPU:
the product's camera_pose_from_spherical / camera_pose_to_spherical against
the oracle, and the oracle's own track_camera on a tiny orbit sequence."""
import numpy as np

from oracle import pyoracle as O
from paper_2312_08715_b200 import b3d, configs


def test_camera_pose_from_spherical_matches_oracle_bitwise():
    rng = np.random.Generator(np.random.PCG64(3))
    for _ in range(500):
        d = rng.uniform(0.2, 3.0)
        az = rng.uniform(-7.0, 7.0)
        alt = rng.uniform(1e-3, np.pi / 2 - 1e-3)
        np.testing.assert_array_equal(b3d.camera_pose_from_spherical(d, az, alt),
                                      O.camera_pose_from_spherical(d, az, alt))


def test_camera_pose_to_spherical_round_trip_and_rejections():
    rng = np.random.Generator(np.random.PCG64(4))
    for _ in range(200):
        d, az, alt = rng.uniform(0.2, 3.0), rng.uniform(0, 2 * np.pi), rng.uniform(0.05, 1.5)
        p = b3d.camera_pose_from_spherical(d, az, alt)
        got = b3d.camera_pose_to_spherical(p)
        assert got is not None and got == O.camera_pose_to_spherical(p)
        assert abs(got[0] - d) < 1e-12 and abs(got[2] - alt) < 1e-9
        assert abs(np.angle(np.exp(1j * (got[1] - az)))) < 1e-9
    # a camera not looking at the origin, and one below the table plane
    p = b3d.camera_pose_from_spherical(1.0, 0.3, 0.4)
    q = p.copy()
    q[4] += 0.01
    assert b3d.camera_pose_to_spherical(q) is None and O.camera_pose_to_spherical(q) is None
    q = p.copy()
    q[6] = -q[6]
    assert b3d.camera_pose_to_spherical(q) is None and O.camera_pose_to_spherical(q) is None


def _oracle_render_cameras(k, inst, cams):
    return np.stack([O.render(k, inst, camera=c) for c in cams])


def test_oracle_track_camera_follows_a_short_orbit():
    seq = configs.orbit_sequence(_oracle_render_cameras, O.voxel_to_mesh, O.box_mesh,
                                 O.contact_to_pose, res=25, n_frames=40, n_voxels=300)
    cams = [O.camera_pose_from_spherical(seq["distance"], a, seq["altitude"])
            for a in seq["azimuths"][:3]]
    frames = configs.orbit_frames(seq, cams)
    est = O.track_camera(frames, seq["k"], seq["instances"], cams[0], seq["noise"],
                         seq["sigma_max"], seq["window"])
    assert est.shape == (3, 7)
    np.testing.assert_array_equal(est[0], cams[0])
    for f in (1, 2):
        assert np.linalg.norm(est[f][4:] - cams[f][4:]) < 0.05  # within the search extents
