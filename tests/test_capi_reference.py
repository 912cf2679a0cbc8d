"""The product's C ABI returns the reference's status codes and error texts
for the same misuse, and the reference's renders bit for bit through
b3d_render (tests/capi_cases.py; fixture tests/golden/ref_capi.json made
from oracle/_ref/libb3d_ref.so -- the reference's b3d_capi.cpp compiled
unmodified -- by tests/golden/make_ref_golden.py capi).

The CPU test runs every case the product settles before touching a device
(argument, intrinsics, noise, file-format, manifest, scene-JSON and `infer`
schema errors); the GPU test runs all of them, including the empty-render
checks, device-side `infer` validation and whole 3- and 20-child renders.
"""
import ctypes
import json
import os
import sys

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


def _compare(got, want):
    assert set(got) <= set(want), sorted(set(got) - set(want))
    diff = {k: (got[k], want[k]) for k in got if got[k] != want[k]}
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
