"""The oracle's and the product's Rng restatements reproduce the reference
Rng (rng.cpp) bit for bit: golden vectors from the reference's own rng.cpp
(tests/golden/make_rng_golden.py)."""
import json
import os

import numpy as np

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rng_golden.json")))


def _draw(O, case):
    st = O.rng_seed(case["seed"])
    if case["split"]:
        st = O.rng_split(st, *case["keys"])
    n = len(case["values"])
    L = O.lib()
    out = []
    for _ in range(n):
        if case["kind"] == 0:
            out.append(int(L.orc_rng_next_u64(st.ctypes.data)))
        elif case["kind"] == 1:
            out.append(int(np.float64(O.rng_uniform(st)).view(np.uint64)))
        elif case["kind"] == 2:
            out.append(O.rng_uniform_int(st, case["m"]))
        else:
            out.append(int(np.float64(O.rng_normal(st)).view(np.uint64)))
    return out


def test_oracle_rng_matches_reference_golden(oracle):
    for case in GOLD["cases"]:
        assert _draw(oracle, case) == [int(v) for v in case["values"]], case


def test_product_rng_seed_split_matches_oracle(oracle):
    """b3d_rng_seed / b3d_rng_split (host side of the device stream)."""
    from paper_2312_08715_b200 import b3d
    for case in GOLD["cases"]:
        a = b3d.rng_seed(case["seed"])
        b = oracle.rng_seed(case["seed"])
        assert np.array_equal(a, b)
        if case["split"]:
            assert np.array_equal(b3d.rng_split(a, *case["keys"]), oracle.rng_split(b, *case["keys"]))
