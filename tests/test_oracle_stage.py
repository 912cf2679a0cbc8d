"""Stage reduction semantics of the oracle (inference.cpp:16-23,315-353,
tracking.cpp:132-134).  No reference test covers this stage;
these pin the restatement to the reference's code semantics directly."""
import math

import numpy as np


def test_normalize_and_all_neg_inf(oracle):
    p, az = oracle.normalize(np.array([0.0, math.log(3.0)]))
    assert not az and abs(p[0] - 0.25) < 1e-15 and abs(p[1] - 0.75) < 1e-15
    p, az = oracle.normalize(np.array([-np.inf, -np.inf, -np.inf]))
    assert az and np.allclose(p, 1 / 3)


def test_argmax_first_of_ties(oracle):
    assert oracle.argmax(np.array([1.0, 3.0, 3.0, 2.0])) == 1
    assert oracle.argmax(np.array([-np.inf, -np.inf])) == 0


def test_logsumexp(oracle):
    x = np.array([1000.0, 1000.0])
    assert abs(oracle.logsumexp(x) - (1000.0 + math.log(2.0))) < 1e-12
    assert oracle.logsumexp(np.array([-np.inf])) == -np.inf


def test_sample_categorical_inverse_cdf(oracle):
    probs = np.array([0.1, 0.2, 0.3, 0.4])
    st = oracle.rng_seed(11)
    u_st = st.copy()
    u = oracle.rng_uniform(u_st)
    got = oracle.sample_categorical(probs, st)
    assert got == int(np.searchsorted(np.cumsum(probs), u, side="right"))
    # u beyond the rounded total -> last index (inference.cpp:352)
    assert oracle.sample_categorical(np.array([0.0, 0.0]), oracle.rng_seed(1)) == 1


def test_sampling_frequencies(oracle):
    probs = np.array([0.5, 0.25, 0.125, 0.125])
    st = oracle.rng_seed(3)
    counts = np.bincount([oracle.sample_categorical(probs, st) for _ in range(20000)], minlength=4)
    assert np.allclose(counts / 20000, probs, atol=0.01)
