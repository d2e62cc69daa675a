"""The tiling solver's CSP engine (csrc/csp.cpp, C ABI include/flashrnn_csp.h)
against (a) exhaustive enumeration and (b) the reference ConstrINT solver
compiled in place (oracle/_ref/libref_csp.so: /root/reference/proj/core/src/csp,
src/plan), on random problems and on the reference planner's own tiling CSPs
(planner.cpp:100-231 build_csp, H100 preset).

The solver returns the FIRST solution in heuristic order (solver.hpp:14-19):
for a sound propagator that is the lexicographically extremal solution under
(order, value preference), so all three must agree exactly.
"""
import ctypes as C
import os
import random

import pytest

from paper_2412_07752_b200.abi import csp_brute_force, csp_solve

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "libref_csp.so")


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/libref_csp.so not built (needs /root/reference)")
    L = C.CDLL(REF)
    L.ref_csp_solve.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_int64)]
    L.ref_csp_brute_count.argtypes = [C.c_char_p, C.c_int64]
    L.ref_csp_brute_count.restype = C.c_int64
    L.ref_build_csp.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int,
                                C.c_int64, C.c_char_p, C.c_size_t]
    return L


def ref_solve(L, text):
    buf = C.create_string_buffer(1 << 20)
    n = C.c_int64()
    rc = L.ref_csp_solve(text.encode(), buf, len(buf), C.byref(n))
    assert rc >= 0, "reference solver error"
    if rc == 0:
        return None
    return dict((k, int(v)) for k, v in (ln.split("=") for ln in buf.value.decode().strip().splitlines()))


def ref_build(L, gpu, ns, ng, dh, nh, batch, dtype, pas, budget=-1):
    buf = C.create_string_buffer(1 << 20)
    assert L.ref_build_csp(gpu.encode(), ns, ng, dh, nh, batch, dtype.encode(), pas, budget, buf, len(buf)) == 0
    return buf.value.decode()


# ---------------------------------------------------------- random problems
def random_problem(rng: random.Random):
    """Small random CSP in text form + its (variable ids, heuristic key)."""
    lines, ids, nodes = [], [], 0
    nres = rng.randint(2, 4)
    for i in range(nres):
        kind = rng.choice(["r", "s", "e"])
        if kind == "r":
            lo = rng.randint(1, 6)
            dom = f"r {lo} {lo + rng.randint(0, 14)}"
        elif kind == "s":
            lo, st = rng.randint(1, 8), rng.randint(2, 5)
            dom = f"s {lo} {lo + st * rng.randint(0, 6)} {st}"
        else:
            dom = "e " + " ".join(str(v) for v in sorted(rng.sample(range(1, 40), rng.randint(1, 6))))
        lines.append(f"v x{i} R {dom}")
        ids.append(f"x{i}")
    consts = {}

    def const(c):
        if c not in consts:
            consts[c] = len(lines)
            lines.append(f"v k{c} C r {c} {c}")
        return consts[c]

    node_lines = []

    def leaf(v):
        nonlocal nodes
        node_lines.append(f"n v {v}")
        nodes += 1
        return nodes - 1

    def expr(depth=0):
        nonlocal nodes
        r = rng.random()
        if depth >= 2 or r < 0.45:
            return leaf(rng.randrange(nres)) if rng.random() < 0.8 else leaf(const(rng.randint(1, 12)))
        a, b = expr(depth + 1), expr(depth + 1)
        node_lines.append(f"n {rng.choice('+*')} {a} {b}")
        nodes += 1
        return nodes - 1

    con_lines = []
    for _ in range(rng.randint(1, 4)):
        a, b = expr(), expr()
        con_lines.append(f"c {rng.choice(['=', '<', '<', '|'])} {a} {b}")
    order = list(range(nres))
    rng.shuffle(order)
    order = order[: rng.randint(0, nres)]
    prefs = {v: rng.choice("SL") for v in order}
    text = "\n".join(lines + node_lines + con_lines + [f"h {v} {prefs[v]}" for v in order]) + "\n"
    full = order + [v for v in range(nres) if v not in order]

    def key(sol):
        return tuple(sol[f"x{v}"] * (-1 if prefs.get(v, "S") == "L" else 1) for v in full)

    return text, key


def test_random_problems_match_brute_force_and_reference(ref):
    rng = random.Random(1234)
    feasible = 0
    for trial in range(400):
        text, key = random_problem(rng)
        mine, _ = csp_solve(text)
        sols = csp_brute_force(text)
        expect = min(sols, key=key) if sols else None
        assert mine == expect, f"trial {trial}: mine {mine} brute {expect}\n{text}"
        assert ref.ref_csp_brute_count(text.encode(), 1 << 22) == len(sols), f"trial {trial}: solution count"
        assert ref_solve(ref, text) == expect, f"trial {trial}: reference disagrees\n{text}"
        feasible += expect is not None
    assert 40 < feasible < 400  # the generator exercises both outcomes


def test_random_problems_without_reference():
    rng = random.Random(99)
    for trial in range(200):
        text, key = random_problem(rng)
        mine, _ = csp_solve(text)
        sols = csp_brute_force(text)
        assert mine == (min(sols, key=key) if sols else None), text


# -------------------------------------------- the reference planner's CSPs
@pytest.mark.parametrize("ns,ng,dh,nh,batch,pas", [
    (2, 4, 64, 1, 16, 0),     # LSTM small head
    (2, 4, 64, 12, 16, 1),    # LSTM NH=12 backward
    (2, 4, 192, 4, 16, 0),    # LSTM NH=4 (config 3)
    (1, 1, 256, 1, 8, 1),     # Elman
])
def test_reference_planner_csps_same_solution(ref, ns, ng, dh, nh, batch, pas):
    text = ref_build(ref, "H100", ns, ng, dh, nh, batch, "bf16", pas)
    mine, st = csp_solve(text)
    theirs = ref_solve(ref, text)
    assert mine == theirs, (mine, theirs)
    print(f"H100 ns={ns} ng={ng} dh={dh} nh={nh} pass={pas}: {mine}  ({st['solve_us']:.0f} us, {st['nodes']} nodes)")


def test_reference_planner_lstm768(ref):
    """The paper's headline shape (LSTM, DH=768): the reference planner's
    forward CSP (SURVEY 8a probe: G[E8 W3 Bk128] S[E16 W2 L24])."""
    text = ref_build(ref, "H100", 2, 4, 768, 1, 16, "bf16", 0)
    mine, st = csp_solve(text)
    assert mine == ref_solve(ref, text)
    assert (mine["E_G"], mine["W_G"], mine["B_G"]) == (8, 3, 128)
    assert st["solve_us"] < 1e6


def test_infeasible_and_malformed():
    assert csp_solve("v a R r 1 3\nv b R r 5 9\nn v 0\nn v 1\nc = 0 1\n")[0] is None
    from paper_2412_07752_b200 import FrnnError
    with pytest.raises(FrnnError):
        csp_solve("v a R r 0 3\n")  # domain values must be >= 1
    with pytest.raises(FrnnError):
        csp_solve("v a R r 1 3\nh 0 L\nh 0 S\n")  # variable listed twice


def test_divisibility_and_progression_domains():
    # a in multiples of 3, a*b == 96, a <= b, 4 | b; largest a first:
    # a=24 -> b=4 (a > b), a=12 -> b=8 (a > b), a=6 -> b=16 ok
    t = ("v a R s 3 30 3\nv b R r 1 100\nv k C r 96 96\nv f C r 4 4\n"
         "n v 0\nn v 1\nn v 2\nn * 0 1\nn v 3\nc = 3 2\nc < 0 1\nc | 4 1\nh 0 L\n")
    sol, _ = csp_solve(t)
    assert sol == {"a": 6, "b": 16}
    # a*a == b with no a | ... : infeasible when b is prime
    assert csp_solve("v a R r 1 50\nv b C r 97 97\nn v 0\nn v 1\nn * 0 0\nc = 2 1\n")[0] is None
    assert csp_solve("v a R r 1 50\nv b C r 49 49\nn v 0\nn v 1\nn * 0 0\nc = 2 1\n")[0] == {"a": 7}


# ------------------------------------ the B200 planner's own tiling CSPs ----
def plan_csp(variant, B, NH, DH, pas, algo):
    from paper_2412_07752_b200.abi import Shape, cell_spec, load
    L = load()
    L.frnn_debug_plan_csp.argtypes = [C.c_void_p, Shape, C.c_int32, C.c_int32, C.c_int32, C.c_char_p, C.c_size_t]
    buf = C.create_string_buffer(1 << 20)
    cell = cell_spec(variant)
    assert L.frnn_debug_plan_csp(C.byref(cell), Shape(1024, B, NH, DH), 1, pas, algo, buf, len(buf)) == 0
    return buf.value.decode()


@pytest.mark.parametrize("variant,B,NH,DH,pas,algo", [
    ("slstm", 16, 1, 768, 0, 1), ("slstm", 16, 1, 768, 1, 1),   # config 2, cluster-resident kernels
    ("lstm", 16, 12, 64, 1, 1), ("lstm", 16, 4, 192, 0, 1),     # config 3
    ("gru", 16, 1, 768, 1, 1),                                  # config 4
    ("slstm", 64, 1, 3072, 0, 2), ("slstm", 64, 1, 3072, 1, 2),  # config 5, alternating path
])
def test_b200_planner_csp_matches_reference_solver(ref, variant, B, NH, DH, pas, algo):
    """The B200 formulation (planner.cpp) solved by the reference ConstrINT
    solver gives the tiling the planner chose."""
    from paper_2412_07752_b200.abi import plan as frnn_plan
    text = plan_csp(variant, B, NH, DH, pas, algo)
    mine, st = csp_solve(text)
    assert mine is not None
    assert ref_solve(ref, text) == mine
    plan = frnn_plan(variant, 1024, B, NH, DH, "bf16", ["forward", "backward"][pas])
    if algo == 1:
        ngp = 1 if variant == "elman" else 4
        assert (plan["ctas_per_group"], plan["rows_per_cta"]) == (mine["CL"], mine["UPC"] * ngp)
    else:
        assert plan["batch_tile"] == mine["N"] and plan["k_split"] == mine.get("KS", 1)
    print(variant, DH, pas, mine, f"{st['solve_us']:.0f} us")
