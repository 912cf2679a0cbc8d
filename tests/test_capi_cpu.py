"""C ABI checks that need no GPU: the library loads, exports exactly what
include/b3d_b200.h declares, host-side entry points work, and GPU entry points
fail cleanly (status + thread-local message, no crash) without a device."""
import ctypes as C

import numpy as np
import pytest

from paper_2312_08715_b200 import b3d


def test_library_exports_every_declared_symbol():
    L = b3d.lib()
    declared = b3d.exported_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name


def test_version_and_depth_image_roundtrip():
    L = b3d.lib()
    assert L.b3d_version().decode().startswith("0.1")
    img = np.arange(12, dtype=np.float32).reshape(3, 4)
    h = C.c_void_p()
    assert L.b3d_depth_image_create(4, 3, img.ctypes.data, C.byref(h)) == 0
    assert L.b3d_depth_image_width(h) == 4 and L.b3d_depth_image_height(h) == 3
    data = np.ctypeslib.as_array(C.cast(L.b3d_depth_image_data(h), C.POINTER(C.c_float)), (12,))
    assert np.array_equal(data, img.ravel())
    L.b3d_depth_image_destroy(h)
    # bad arguments -> B3D_ERROR with the reference's message
    assert L.b3d_depth_image_create(0, 3, img.ctypes.data, C.byref(h)) == 1
    assert L.b3d_last_error().decode() == "bad arguments"


def test_gpu_entry_points_fail_cleanly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = b3d.lib()
    h = C.c_void_p()
    st = L.b3d_gpu_context_create(0, C.byref(h))
    assert st != 0 and L.b3d_last_error()


def test_voxel_to_mesh_errors():
    L = b3d.lib()
    nv, nt = C.c_uint64(), C.c_uint64()
    o = np.zeros(3)
    buf = np.zeros(24)
    tb = np.zeros(36, dtype=np.uint32)
    vox = np.zeros((0, 3), dtype=np.int32)
    st = L.b3d_voxel_to_mesh(vox.ctypes.data, 0, 0.1, o.ctypes.data, buf.ctypes.data,
                             tb.ctypes.data, C.byref(nv), C.byref(nt))
    assert st == 1 and b"empty grid" in L.b3d_last_error()


def test_mesh_cull_sign_closed_open_and_flipped():
    """Back-face culling is enabled only for closed meshes (every directed edge
    matched by its reverse); the sign follows the winding (enclosed volume)."""
    from paper_2312_08715_b200 import synth
    for vox in (synth.eden_blob(300, 4), synth.random_walk_blob(300, 5)):
        v, t = b3d.voxel_to_mesh(vox, 0.005, np.zeros(3))
        s = b3d.mesh_cull_sign(v, t)
        assert s == 1  # voxel_to_mesh winds faces outward (geometry.cpp:142-177)
        assert b3d.mesh_cull_sign(v, t[:, ::-1]) == -1
        assert b3d.mesh_cull_sign(v, t[1:]) == 0      # a hole
        t2 = t.copy()
        t2[0] = t2[0, [0, 0, 1]]                       # degenerate index
        assert b3d.mesh_cull_sign(v, t2) == 0
    # the reference box mesh is closed too; a lone triangle is not
    from oracle import pyoracle as O
    bv, bt = O.box_mesh([-0.05, -0.04, 0.0], [0.05, 0.04, 0.09])
    assert b3d.mesh_cull_sign(bv, bt) in (1, -1)
    assert b3d.mesh_cull_sign(bv, bt[:1]) == 0


def test_box_mesh_and_contact_to_pose_match_oracle_bitwise():
    """Host scene-graph helpers of the product (make_box_mesh,
    contact_to_pose) against the oracle restatement."""
    from oracle import pyoracle as O
    from paper_2312_08715_b200 import synth
    lo, hi = np.array([-0.25, -0.2, -0.01]), np.array([0.25, 0.2, 0.0])
    v1, t1 = b3d.box_mesh(lo, hi)
    v2, t2 = O.box_mesh(lo, hi)
    np.testing.assert_array_equal(v1, v2)
    np.testing.assert_array_equal(t1, t2)
    assert b3d.mesh_cull_sign(v1, t1) == 1
    v, t = b3d.voxel_to_mesh(synth.eden_blob(400, 2), 0.005, np.zeros(3))
    amin, amax = v.min(axis=0), v.max(axis=0)
    rng = np.random.Generator(np.random.PCG64(6))
    for face in range(1, 7):
        for _ in range(30):
            dx, dy, th = rng.uniform(0, 0.3), rng.uniform(0, 0.3), rng.uniform(0, 6.28)
            np.testing.assert_array_equal(b3d.contact_to_pose(0.5, 0.5, amin, amax, face, dx, dy, th),
                                          O.contact_to_pose(0.5, 0.5, amin, amax, face, dx, dy, th))
    with pytest.raises(b3d.B3DError):
        b3d.contact_to_pose(0.5, 0.5, amin, amax, 1, 0.49, 0.1, 0.0)


def test_buffer_pointers_match_numpy():
    """b3d._ptr (the wrapper's per-call pointer path) returns the array's data
    address for writable, read-only, sliced, empty and non-float arrays."""
    a = np.arange(12.0).reshape(3, 4)
    assert b3d._ptr(a) == a.ctypes.data
    assert b3d._ptr(a[1:]) == a[1:].ctypes.data
    r = np.zeros(4, dtype=np.uint64)
    r.flags.writeable = False
    assert b3d._ptr(r) == r.ctypes.data
    e = np.zeros(0)
    assert b3d._ptr(e) == e.ctypes.data
    u8 = np.zeros(5, dtype=np.uint8)
    assert b3d._ptr(u8) == u8.ctypes.data
    assert b3d._ptr(None) is None
    with pytest.raises(ValueError):
        b3d._ptr(a[:, ::2])
