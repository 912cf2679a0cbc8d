"""The reference's handle API (b3d.h: models, libraries, scenes, SDPT/SVOX
files, b3d_infer's strict config) on CPU -- everything up to the device
work."""
import json

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2312_08715_b200 import b3d, synth


def _model(n=200, seed=3, id_=0, res=0.005, origin=(-0.03, -0.02, 0.0)):
    vox = synth.eden_blob(n, seed)
    return vox, b3d.Model.from_voxels(vox, res, np.array(origin), id_)


def test_model_from_voxels_matches_voxel_to_mesh_and_bounds():
    vox, m = _model()
    v, t = m.mesh()
    ov, ot = O.voxel_to_mesh(vox, 0.005, np.array([-0.03, -0.02, 0.0]))
    np.testing.assert_array_equal(v, ov)
    np.testing.assert_array_equal(t, ot)
    np.testing.assert_array_equal(m.bbox(), v.max(axis=0) - v.min(axis=0))
    assert m.voxel_count() == vox.shape[0] and m.resolution() == 0.005


def test_svox_and_sdpt_round_trips(tmp_path):
    """SVOX stores resolution / origin as float32 and voxels in stored order
    (io.cpp:118-147); SDPT is raw float32 (io.cpp:91-116)."""
    vox, m = _model(res=0.25, origin=(-0.25, -0.5, 0.0))  # float32-exact grid
    m.save(tmp_path / "a.svox")
    raw = (tmp_path / "a.svox").read_bytes()
    assert raw[:4] == b"SVOX" and len(raw) == 24 + 12 * vox.shape[0]
    m2 = b3d.Model.load(tmp_path / "a.svox", 0)
    v1, t1 = m.mesh()
    v2, t2 = m2.mesh()
    np.testing.assert_array_equal(v1, v2)
    np.testing.assert_array_equal(t1, t2)
    d = np.random.Generator(np.random.PCG64(1)).uniform(0.1, 5, size=(7, 9)).astype(np.float32)
    b3d.depth_image_save(d, tmp_path / "d.sdpt")
    assert (tmp_path / "d.sdpt").read_bytes()[:4] == b"SDPT"
    np.testing.assert_array_equal(b3d.depth_image_load(tmp_path / "d.sdpt"), d)
    (tmp_path / "bad.sdpt").write_bytes(b"SDPX" + bytes(8))
    with pytest.raises(b3d.B3DError) as e:
        b3d.depth_image_load(tmp_path / "bad.sdpt")
    assert e.value.status == b3d.B3D_ERROR_IO and "bad magic bytes" in str(e.value)


def test_library_manifest_and_scene_json(tmp_path):
    _, m0 = _model(150, 1, 0)
    _, m1 = _model(250, 2, 1)
    m0.save(tmp_path / "m0.svox")
    m1.save(tmp_path / "m1.svox")
    (tmp_path / "lib.json").write_text(json.dumps(
        {"models": [{"id": 1, "path": "m1.svox"}, {"id": 0, "path": "m0.svox"}]}))
    lib = b3d.Library.open(tmp_path / "lib.json")
    assert len(lib) == 2
    sc = b3d.Scene.from_json(json.dumps({"table": {"width": 0.5, "height": 0.4},
                                         "children": [{"object_id": 1, "face": 2, "dx": 0.1,
                                                       "dy": 0.05, "dtheta": 1.25}]}), lib)
    back = json.loads(sc.to_json())
    assert back["table"] == {"width": 0.5, "height": 0.4, "thickness": 0.01}
    assert back["children"] == [{"object_id": 1, "face": 2, "dx": 0.1, "dy": 0.05,
                                 "dtheta": 1.25}]
    with pytest.raises(b3d.B3DError) as e:
        b3d.Scene.from_json('{"children": []}', lib)
    assert e.value.status == b3d.B3D_ERROR_CONFIG and "missing 'table'" in str(e.value)
    with pytest.raises(b3d.B3DError) as e:
        b3d.Scene.from_json('{"table": {"width": 1, "height": 1}, "children": '
                            '[{"object_id": 5, "face": 1, "dx": 0, "dy": 0, "dtheta": 0}]}', lib)
    assert "object_id out of library range" in str(e.value)


def test_infer_config_is_strict_like_the_reference():
    """ConfigReader semantics (config.cpp): unknown keys, missing required
    keys and wrong types are B3D_ERROR_CONFIG -- reported before any device
    work."""
    _, m0 = _model()
    lib = b3d.Library.create([m0])
    obs = np.full((4, 4), 5.0, dtype=np.float32)
    cam = [1.0, 0, 0, 0, 0, 0, 0]
    intr = {"fx": 4, "fy": 4, "cx": 2, "cy": 2, "width": 4, "height": 4, "near": 0.1, "far": 5}
    cases = [
        ("{}", "b3d_infer: config requires 'intrinsics'"),
        (json.dumps({"intrinsics": intr}), "b3d_infer config: missing required key 'table'"),
        (json.dumps({"intrinsics": intr, "table": {"width": 1, "height": 1}, "bogus": 1}),
         "b3d_infer config: unknown key 'bogus'"),
        (json.dumps({"intrinsics": {**intr, "extra": 1}, "table": {"width": 1, "height": 1}}),
         "b3d_infer config.intrinsics: unknown key 'extra'"),
        (json.dumps({"intrinsics": intr, "table": {"width": 1, "height": 1},
                     "particles": "many"}), "b3d_infer config: key 'particles' has the wrong type"),
        ("{not json", "invalid inference config JSON"),
    ]
    for cfg, msg in cases:
        with pytest.raises(b3d.B3DError) as e:
            b3d.infer(obs, cam, lib, cfg, 0)
        assert e.value.status == b3d.B3D_ERROR_CONFIG and str(e.value).endswith(msg), str(e.value)
