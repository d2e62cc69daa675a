import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    import oracle as O
    return O.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle as O
    if not O.Reference.available():
        pytest.skip("reference engine (oracle/_ref/libref.so) not built")
    return O.Reference()


def normwise(a, b):
    """||a - b|| / ||b|| (b = oracle); 0 when both vanish."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    na = np.linalg.norm(a - b)
    if nb == 0:
        return na
    return na / nb


def rel_floor(a, b, floor):
    """max |a-b| / max(|a|,|b|,floor) -- the form of gradcheck.cpp:11-14."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))


def trace_control(orc, v, R, states, gates, dsf, target_err, realizations=8, clip="off", mag=0.0,
                  dh=None, seed=0):
    """Sensitivity of the f64 backward (engine.hpp:221-339) to a bf16-level
    change of its trace -- the CONTROL the sLSTM end-to-end gradient bound is
    tied to.  The trace (states, gates of the f64 oracle forward) is perturbed
    multiplicatively and rounded to bf16 (scalar.hpp:20-27) so that its
    normwise distance from the f64 trace equals ``target_err`` (the GPU
    forward's measured trace error; plain rounding when that is smaller), and
    the oracle backward on each perturbed trace is compared with the one on
    the f64 trace.  Returns {grad: max over realizations} and the per-
    realization list.  Smooth cells give ~1e-3; sLSTM's Jacobian switches
    branch at the stabiliser tie (cell.hpp:153), so near-tie elements flip and
    the spread over realizations is wide at small T (few elements)."""
    exact = orc.backward(v, R, states, gates, dsf, clip, mag, dh)
    base = max(normwise(orc.round_bf16(states), states), 1e-30)
    sc = float(np.sqrt(max(target_err ** 2 - base ** 2, 0.0)))
    rs = np.random.RandomState(seed)
    runs = []
    for k in range(realizations):
        noise = sc if k else 0.0  # realization 0: plain bf16 rounding
        st = orc.round_bf16(states * (1 + noise * rs.standard_normal(states.shape)))
        ga = orc.round_bf16(gates * (1 + noise * rs.standard_normal(gates.shape)))
        g = orc.backward(v, R, st, ga, dsf, clip, mag, dh)
        runs.append({key: normwise(g[key], exact[key]) for key in exact})
    return {key: max(r[key] for r in runs) for key in exact}, runs
