"""The product's C ABI returns the reference's status codes and error texts
for the same misuse, and the reference's renders bit for bit through
b3d_render (tests/capi_cases.py; fixture tests/golden/ref_capi.json made
from oracle/_ref/libb3d_ref.so -- the reference's b3d_capi.cpp compiled
unmodified -- by tests/golden/make_ref_golden.py capi).

The CPU test runs every case the product settles before touching a device
(argument, intrinsics, noise, file-format, manifest, scene-JSON and `infer`
schema errors); the GPU test runs all of them, including the empty-render
checks, device-side `infer` validation, whole 3- and 20-child renders and
`infer` runs placing ten objects and one (draws equal, log evidence to 1e-6
relative, type marginal and MAP pose, the accessors' errors).
"""
import ctypes
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import capi_cases  # noqa: E402

from paper_2312_08715_b200 import b3d  # noqa: E402


def _fixture():
    with open(os.path.join(HERE, "golden", "ref_capi.json")) as f:
        return json.load(f)


def _lib():
    # a private ctypes handle on the same loaded library: capi_cases sets its
    # own argtypes, which must not leak into b3d.py's bindings
    return ctypes.CDLL(b3d.lib()._name)


def _same(a, b):
    if isinstance(b[1], dict):  # an inference result: draws equal, evidence to 1e-6
        if a[0] != b[0] or not isinstance(a[1], dict):
            return False
        ga, wa = a[1], b[1]
        if abs(ga["log_evidence"] - wa["log_evidence"]) > 1e-6 * abs(wa["log_evidence"]):
            return False
        if set(ga) != set(wa):
            return False
        # the marginal is a sum of exp(log weight - lse): a weight's absolute
        # error (scores ~4e3 at ~3e-8 relative) moves it by ~1e-6 relative
        if "marginal" in wa and not np.allclose(ga["marginal"], wa["marginal"], rtol=1e-4,
                                                atol=1e-9):
            return False
        if "map_pose" in wa and not np.allclose(ga["map_pose"], wa["map_pose"], rtol=0,
                                                atol=1e-12):
            return False
        return len(ga["particles"]) == len(wa["particles"]) and all(
            len(p) == len(q) and all(x[:2] == y[:2] and np.allclose(x[2:], y[2:], rtol=0,
                                                                    atol=1e-12)
                                     for x, y in zip(p, q))
            for p, q in zip(ga["particles"], wa["particles"]))
    return a == b


def _compare(got, want):
    assert set(got) <= set(want), sorted(set(got) - set(want))
    diff = {k: (got[k], want[k]) for k in got if not _same(got[k], want[k])}
    assert not diff, json.dumps(diff, indent=1)


def test_capi_errors_match_reference_cpu():
    got = capi_cases.run_cases(_lib(), gpu=False)
    assert len(got) >= 30
    _compare(got, _fixture())


@pytest.mark.gpu
def test_capi_errors_and_renders_match_reference_gpu():
    want = _fixture()
    got = capi_cases.run_cases(_lib(), gpu=True)
    assert set(got) == set(want)
    _compare(got, want)


def _fuzz():
    with open(os.path.join(HERE, "golden", "ref_infer_fuzz.json")) as f:
        return json.load(f)


def _device_error(res):
    return res[0] != 0 and "cuda" in res[1].lower()


def test_infer_config_fuzz_cpu():
    """240 seeded random b3d_infer configurations plus 200 character-level
    edits of one (tests/infer_fuzz.py; strings, escapes, surrogates, control
    characters, numbers, BOM, repeated keys -- the JSON parser's verdicts): every
    one the product settles on the host -- JSON and schema errors, nlohmann's
    number conversions (booleans and floats into integers, wrapping, gcc's
    right-to-left argument order), make_inference_context / run_smc checks
    in the reference's order -- gives the reference's status and text."""
    import infer_fuzz
    cases = _fuzz()
    got = infer_fuzz.run(_lib(), [c["config"] for c in cases], False)
    compared = 0
    for c, g in zip(cases, got):
        if _device_error(g):
            continue  # needs the device: the GPU test covers it
        compared += 1
        assert _same(g, c["result"]), (c["config"], g, c["result"])
    assert compared >= 380


@pytest.mark.gpu
def test_infer_config_fuzz_gpu():
    """All 240, including the valid ones (particles and evidence) and the
    errors the inference itself raises (empty renders, all-zero stage 0)."""
    import infer_fuzz
    cases = _fuzz()
    got = infer_fuzz.run(_lib(), [c["config"] for c in cases], True)
    for c, g in zip(cases, got):
        assert _same(g, c["result"]), (c["config"], g, c["result"])


def test_scene_json_fuzz():
    """200 seeded random scene documents through b3d_scene_from_json and back
    through b3d_scene_to_json: the reference's status and message, or its
    exact output text (nlohmann's number format)."""
    import infer_fuzz
    with open(os.path.join(HERE, "golden", "ref_scene_fuzz.json")) as f:
        cases = json.load(f)
    got = infer_fuzz.run_scenes(_lib(), [c["scene"] for c in cases])
    for c, g in zip(cases, got):
        assert g == c["result"], (c["scene"], g, c["result"])


def test_file_format_fuzz():
    """200 seeded random SDPT / SVOX files (byte flips, cuts, edited headers
    and payloads): the reference's status and message, or the same image
    (dims + float bytes) / the same model re-saved byte for byte."""
    import base64
    import infer_fuzz
    with open(os.path.join(HERE, "golden", "ref_file_fuzz.json")) as f:
        cases = json.load(f)
    got = infer_fuzz.run_files(_lib(), [(c["kind"], base64.b64decode(c["bytes"]))
                                        for c in cases])
    for c, g in zip(cases, got):
        assert g == c["result"], (c["kind"], c["bytes"], g, c["result"])


def test_manifest_fuzz():
    """150 seeded random library manifests: the reference's status and
    message (nlohmann's own exception texts included), or the same library size."""
    import infer_fuzz
    with open(os.path.join(HERE, "golden", "ref_manifest_fuzz.json")) as f:
        cases = json.load(f)
    got = infer_fuzz.run_manifests(_lib(), [c["manifest"] for c in cases])
    for c, g in zip(cases, got):
        assert g == c["result"], (c["manifest"], g, c["result"])


def _check_calls(name, gpu):
    import infer_fuzz
    with open(os.path.join(HERE, "golden", f"ref_{name}_fuzz.json")) as f:
        cases = json.load(f)
    run = infer_fuzz.run_loglik if name == "loglik" else infer_fuzz.run_render
    got = run(_lib(), [c["case"] for c in cases])
    compared = 0
    for c, g in zip(cases, got):
        want = c["result"]
        if not gpu and _device_error(g):
            continue
        compared += 1
        if name == "loglik" and want[0] == 0 and g[0] == 0 and g[1] != want[1]:
            # the windowed / full likelihood on the device in fp64 (equal
            # infinities compare equal above)
            assert abs(g[1] - want[1]) <= 1e-9 * abs(want[1]), (c["case"], g, want)
        else:
            assert g == want, (c["case"], g, want)
    return compared


def test_loglik_and_render_fuzz_cpu():
    """160 random b3d_log_likelihood calls (sizes, sentinel fractions,
    intrinsics, noise, windows) and 120 random b3d_render calls (scenes of up
    to 18 children, invalid contacts and faces, non-unit cameras, invalid
    intrinsics): every error the product raises before the device equals the
    reference's, in the reference's order of checks."""
    assert _check_calls("loglik", False) >= 140
    assert _check_calls("render", False) >= 90


@pytest.mark.gpu
def test_loglik_and_render_fuzz_gpu():
    """All of them: values within 1e-9 relative, renders bitwise (sha256)."""
    assert _check_calls("loglik", True) == 160
    assert _check_calls("render", True) == 120
