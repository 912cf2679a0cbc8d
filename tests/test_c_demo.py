"""A C program written against the reference's public API (examples/
infer_demo.c) compiles against include/b3d_b200.h and links, unchanged,
against this library -- and, where the reference library was built here
(oracle/_ref), against the reference's own: same output for the same files."""
import json
import os
import shutil
import struct
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_DIR = os.path.join(ROOT, "paper_2312_08715_b200", "_lib")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libb3d_ref.so")


def _build(tmp, against_ref=False):
    exe = os.path.join(tmp, "demo_ref" if against_ref else "demo")
    if against_ref:
        libs = [REF_LIB, f"-Wl,-rpath,{os.path.dirname(REF_LIB)}"]
    else:
        libs = [f"-L{LIB_DIR}", "-lb3d_b200", f"-Wl,-rpath,{LIB_DIR}"]
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I",
                    os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "infer_demo.c"),
                    "-o", exe] + libs, check=True, capture_output=True, text=True)
    return exe


def _world(tmp):
    v = np.array([[0, 0, 0], [1, 0, 0]], dtype="<i4")
    with open(os.path.join(tmp, "a.svox"), "wb") as f:
        f.write(b"SVOX" + struct.pack("<4f", 0.01, 0, 0, 0) + struct.pack("<I", 2) + v.tobytes())
    with open(os.path.join(tmp, "m.json"), "w") as f:
        json.dump({"models": [{"id": 0, "path": "a.svox"}]}, f)
    d = np.full((12, 16), 0.5, dtype="<f4")
    d[4:8, 6:10] = 0.48
    with open(os.path.join(tmp, "obs.sdpt"), "wb") as f:
        f.write(b"SDPT" + struct.pack("<II", 16, 12) + d.tobytes())
    return {"intrinsics": {"fx": 20.0, "fy": 20.0, "cx": 7.5, "cy": 5.5, "width": 16,
                           "height": 12, "near": 0.05, "far": 4.0},
            "table": {"width": 0.2, "height": 0.2},
            "schedule": {"stage0": [1, 1, 2], "refine": [[1, 1, 2]]},
            "noise_grid": {"p_outlier": [0.1], "sigma": [0.02]}, "particles": 3}


def _run(exe, tmp, *args):
    r = subprocess.run([exe] + list(args), capture_output=True, text=True, cwd=tmp, timeout=300)
    return r.returncode, r.stdout.replace(tmp, "<tmp>")


ERROR_CASES = [
    ("none.json", "obs.sdpt", "{}"),
    ("m.json", "none.sdpt", "{}"),
    ("m.json", "obs.sdpt", "{bad json"),
    ("m.json", "obs.sdpt", json.dumps({"table": {"width": 1, "height": 1}})),
    ("m.json", "obs.sdpt", "CFG_BOGUS"),
]


def _args(tmp, cfg, a):
    man, obs, text = a
    if text == "CFG_BOGUS":
        text = json.dumps(dict(cfg, bogus=1))
    return os.path.join(tmp, man), os.path.join(tmp, obs), text


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no C compiler")
def test_c_program_links_and_reports_errors():
    tmp = tempfile.mkdtemp()
    cfg = _world(tmp)
    exe = _build(tmp)
    ref = _build(tmp, True) if os.path.exists(REF_LIB) else None
    for a in ERROR_CASES:
        rc, out = _run(exe, tmp, *_args(tmp, cfg, a))
        assert rc == 1 and "status" in out, out
        if ref:
            assert (rc, out) == _run(ref, tmp, *_args(tmp, cfg, a)), a


@pytest.mark.gpu
def test_c_program_full_inference():
    tmp = tempfile.mkdtemp()
    cfg = _world(tmp)
    exe = _build(tmp)
    rc, out = _run(exe, tmp, os.path.join(tmp, "m.json"), os.path.join(tmp, "obs.sdpt"),
                   json.dumps(cfg), "3")
    assert rc == 0, out
    lines = out.splitlines()
    assert lines[0].startswith("particles 3 log_evidence")
    assert len([ln for ln in lines if ln.startswith("{")]) == 3


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="reference library not built")
def test_c_program_same_output_as_the_reference_library():
    """The same C program and files through both libraries: every particle's
    children print identically (the same draws, nlohmann's number format),
    the evidence agrees to 1e-6 relative."""
    tmp = tempfile.mkdtemp()
    cfg = _world(tmp)
    args = (os.path.join(tmp, "m.json"), os.path.join(tmp, "obs.sdpt"), json.dumps(cfg), "3")
    rc, out = _run(_build(tmp), tmp, *args)
    rc_r, out_r = _run(_build(tmp, True), tmp, *args)
    assert rc == rc_r == 0
    ev = float(out.splitlines()[0].split()[-1])
    ev_r = float(out_r.splitlines()[0].split()[-1])
    assert abs(ev - ev_r) <= 1e-6 * abs(ev_r)
    kids = [ln.split('],"log_weight"')[0] for ln in out.splitlines() if ln.startswith("{")]
    kids_r = [ln.split('],"log_weight"')[0] for ln in out_r.splitlines() if ln.startswith("{")]
    assert kids == kids_r and len(kids) == 3
