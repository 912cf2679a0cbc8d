"""Generates tests/golden/rng_golden.json from the REFERENCE's own RNG
(proj/src/core/rng.cpp compiled into oracle/_ref/libref_rng.so by
`make -C oracle ref`).  Run in the build container (needs /root/reference);
the committed JSON is what the tests read on any machine."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as O  # noqa: E402

CASES = [
    # seed, split, k0, k1, k2, kind (0 u64, 1 uniform bits, 2 uniform_int, 3 normal bits), m, n
    (0, 0, 0, 0, 0, 0, 0, 64),
    (42, 0, 0, 0, 0, 1, 0, 64),
    (7, 1, 3, 0, 0, 0, 0, 32),
    (7, 1, 1, 2, 3, 1, 0, 32),
    (123456789, 1, 0x0F, 5, 0, 2, 1000, 64),
    (99, 0, 0, 0, 0, 2, 6, 64),
    (5, 0, 0, 0, 0, 3, 0, 32),
    (2**63 + 11, 1, 2**40, 17, 9, 0, 0, 16),
]


def main():
    if not O.ref_rng_available():
        raise SystemExit("oracle/_ref/libref_rng.so missing: run make -C oracle ref")
    out = []
    for seed, split, k0, k1, k2, kind, m, n in CASES:
        vals = O.ref_rng_draw(seed, split, k0, k1, k2, kind, m, n)
        out.append({"seed": seed, "split": split, "keys": [k0, k1, k2], "kind": kind, "m": m,
                    "values": [str(int(x)) for x in vals]})
    with open(os.path.join(HERE, "rng_golden.json"), "w") as f:
        json.dump({"source": "reference proj/src/core/rng.cpp via oracle/_ref/libref_rng.so",
                   "cases": out}, f, indent=1)


if __name__ == "__main__":
    main()
