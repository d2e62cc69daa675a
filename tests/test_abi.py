"""CPU tests of the C ABI boundary (no GPU needed, no compute calls).

* libflashrnn.so loads and exports every symbol include/*.h declares;
* argument validation mirrors the reference's std::invalid_argument checks
  (engine.hpp:107, :116-129) and runs before any device work;
* without an sm_100 device the hot path fails loudly (no CPU fallback);
* the tiling planner returns feasible plans for every BASELINE config;
* the batch x head partitioner covers the problem exactly once.
"""
import ctypes as C
import os
import re

import pytest

from paper_2412_07752_b200 import abi
from paper_2412_07752_b200.abi import Cell, Clip, Options, PlanInfo, Shape, cell_spec, load, partition

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    syms = set()
    for h in sorted(f for f in os.listdir(os.path.join(ROOT, "include")) if f.endswith(".h")):
        text = open(os.path.join(ROOT, "include", h)).read()
        syms |= set(re.findall(r"FRNN_API\s+[\w\s\*]*?\b(frnn_\w+)\s*\(", text))
    return syms


def test_library_exports_every_declared_symbol():
    L = load()
    syms = header_symbols()
    assert {"frnn_forward", "frnn_backward", "frnn_plan", "frnn_workspace_size", "frnn_partition"} <= syms
    for s in sorted(syms):
        assert hasattr(L, s), f"missing export {s}"
    out = os.popen(f"nm -D {abi.lib_path()}").read()
    for s in syms:
        assert re.search(rf"\bT {s}\b", out), s


def test_version_and_cell_specs():
    L = load()
    assert b"sm_100a" in L.frnn_version()
    expect = {"elman": (1, 1, [1], [1]), "lstm": (2, 4, [1] * 4, [1] * 4),
              "gru": (1, 4, [1, 1, 0, 1], [1, 1, 1, 0]), "slstm": (4, 4, [1] * 4, [1] * 4)}
    for v, (ns, ng, rec, inp) in expect.items():  # cell.hpp:25-53
        c = cell_spec(v)
        assert (c.num_states, c.num_gates) == (ns, ng)
        assert list(c.uses_recurrent[:ng]) == rec and list(c.uses_input[:ng]) == inp


def _fwd(cell, shape, dtype=1, ptr=256, ws=1 << 30, opts=None):
    L = load()
    p = C.c_void_p(ptr)
    return L.frnn_forward(C.byref(cell), shape, dtype, p, p, p, p, p, p, p, ws, opts, None)


def test_validation_mirrors_reference_errors():
    L = load()
    c = cell_spec("lstm")
    bad = Cell.from_buffer_copy(c)
    bad.num_states = 3  # engine.hpp:119 counts disagree
    assert _fwd(bad, Shape(4, 2, 1, 8)) == 1
    assert b"disagree" in L.frnn_last_error()
    assert _fwd(c, Shape(4, 0, 1, 8)) == 1  # degenerate shape (engine.hpp:121-122)
    assert _fwd(c, Shape(-1, 2, 1, 8)) == 1
    assert _fwd(c, Shape(4, 2, 1, 0)) == 1
    assert _fwd(c, Shape(4, 2, 1, 8), dtype=7) == 3  # unsupported dtype
    assert _fwd(c, Shape(4, 2, 1, 8), ptr=0) == 6  # null tensor
    # clip magnitude must be positive (engine.hpp:107)
    p = C.c_void_p(256)
    rc = L.frnn_backward(C.byref(c), Shape(4, 2, 1, 8), 1, p, p, p, p, p, None, Clip(1, 0.0), p, p, p, p, p,
                         1 << 30, None, None)
    assert rc == 6 and b"positive" in L.frnn_last_error()


def test_misaligned_pointers_rejected():
    """The kernels move rows with 16-byte loads / TMA: a tensor base that is not
    16-byte aligned (e.g. a sliced tensor) is an argument error, checked before
    any device work."""
    L = load()
    c = cell_spec("lstm")
    assert _fwd(c, Shape(4, 2, 1, 8), ptr=256 + 2) == 6
    assert b"16-byte aligned" in L.frnn_last_error()
    p, q = C.c_void_p(256), C.c_void_p(256 + 8)
    rc = L.frnn_backward(C.byref(c), Shape(4, 2, 1, 8), 1, p, p, p, p, p, None, Clip(0, 0.0), p, p, q, p, p,
                         1 << 30, None, None)
    assert rc == 6 and b"dR is not 16-byte aligned" in L.frnn_last_error()


def test_pass_validated():
    L = load()
    info = PlanInfo()
    n = C.c_size_t()
    for bad in (2, -1):
        assert L.frnn_plan(C.byref(cell_spec("lstm")), Shape(8, 4, 1, 64), 1, bad, None, C.byref(info)) == 6
        assert b"pass" in L.frnn_last_error()
        assert L.frnn_workspace_size(C.byref(cell_spec("lstm")), Shape(8, 4, 1, 64), 1, bad, None,
                                     C.byref(n)) == 6


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    rc = _fwd(cell_spec("lstm"), Shape(4, 2, 1, 8))
    assert rc == 5  # FRNN_ECUDA: fails loudly, never computes on the CPU
    assert load().frnn_last_error()


@pytest.mark.parametrize("variant,NH,DH,B,dtype,algo", [
    ("lstm", 1, 64, 8, 0, 3),        # config 1: fp32 -> SIMT FFMA kernels
    ("slstm", 1, 768, 16, 1, 1),     # config 2: fused, cluster-resident
    ("lstm", 4, 192, 16, 1, 1),      # config 3
    ("lstm", 12, 64, 16, 1, 1),
    ("gru", 1, 768, 16, 1, 1),       # config 4
    ("elman", 1, 768, 16, 1, 1),
    ("slstm", 1, 3072, 64, 1, 2),    # config 5: R exceeds on-chip capacity -> alternating
])
def test_planner_configs(variant, NH, DH, B, dtype, algo):
    L = load()
    for ps in (0, 1):
        info = PlanInfo()
        rc = L.frnn_plan(C.byref(cell_spec(variant)), Shape(1024, B, NH, DH), dtype, ps, None, C.byref(info))
        assert rc == 0, L.frnn_last_error()
        assert info.algo == algo
        if algo == 1:
            assert info.cluster >= 1 and info.tmem_cols <= 512 and info.smem_bytes <= 232448
            assert info.cluster <= 16
        n = C.c_size_t()
        assert L.frnn_workspace_size(C.byref(cell_spec(variant)), Shape(1024, B, NH, DH), dtype, ps, None,
                                     C.byref(n)) == 0
        assert n.value >= info.workspace_bytes


def test_forced_algorithm_rejections():
    L = load()
    info = PlanInfo()
    o = Options(0, abi.ALGO["fused"])
    assert L.frnn_plan(C.byref(cell_spec("lstm")), Shape(8, 4, 1, 64), 0, 0, C.byref(o), C.byref(info)) == 3
    o = Options(0, abi.ALGO["simt"])
    assert L.frnn_plan(C.byref(cell_spec("lstm")), Shape(8, 4, 1, 64), 1, 0, C.byref(o), C.byref(info)) == 3


@pytest.mark.parametrize("B,NH,world", [(16, 1, 2), (16, 1, 8), (16, 4, 8), (16, 12, 8), (64, 1, 8), (7, 3, 3)])
def test_partition_covers_exactly_once(B, NH, world):
    seen = {}
    for r in range(world):
        s = partition(64, B, NH, 32, world, r)
        assert 0 <= s["batch_begin"] < s["batch_end"] <= B
        assert 0 <= s["head_begin"] < s["head_end"] <= NH
        for b in range(s["batch_begin"], s["batch_end"]):
            for h in range(s["head_begin"], s["head_end"]):
                seen[(b, h)] = seen.get((b, h), 0) + 1
        # dR/db need a sum across ranks only when the batch is split
        nbatch = len({(partition(64, B, NH, 32, world, q)["batch_begin"]) for q in range(world)})
        assert s["reduce_params"] == (nbatch > 1)
    assert len(seen) == B * NH and set(seen.values()) == {1}


def test_partition_rejects_bad_args():
    with pytest.raises(abi.FrnnError):
        partition(8, 2, 1, 8, 4, 0)  # more batch shards than rows
    with pytest.raises(abi.FrnnError):
        partition(8, 2, 1, 8, 2, 2)  # rank out of range


def test_plan_json_schema():
    from paper_2412_07752_b200.abi import plan_json
    j = plan_json("slstm", 1024, 16, 1, 768, "bf16", "backward")
    assert j["schema_version"] == 1 and j["pass"] == "backward" and j["algo"] == "fused"
    assert j["shape"] == {"num_states": 4, "num_gates": 4, "head_dim": 768, "num_heads": 1, "batch": 16,
                          "seq_len": 1024, "dtype": "bf16"}
    assert j["tiling"]["cluster"] == 16 and j["tiling"]["units_per_cta"] == 48
    assert j["footprint"]["r_matrix_bytes_per_head"] == 4 * 768 * 768 * 2
    k = plan_json("slstm", 1024, 64, 1, 3072, "bf16", "backward")
    assert k["algo"] == "alternating" and k["tiling"]["k_split"] >= 1 and k["tiling"]["stages"] >= 2
    assert k["tiling"]["step_kernels"] == "tcgen05"
    # bf16 head dims the tensor-core kernels cannot tile fall to the FFMA step kernels
    for v, dh in (("lstm", 20), ("gru", 36), ("elman", 1000)):
        f = plan_json(v, 16, 8, 1, dh, "bf16", "forward")
        assert f["algo"] == "alternating" and f["tiling"]["step_kernels"] == "ffma"


# ------------------------------------------- persistent plan cache ----
CACHE_SHAPES = [("slstm", 1024, 16, 1, 768, "bf16", "forward"), ("slstm", 1024, 16, 1, 768, "bf16", "backward"),
                ("lstm", 64, 8, 1, 64, "f32", "forward"), ("slstm", 1024, 64, 1, 3072, "bf16", "backward")]


def test_plan_cache_roundtrip(tmp_path):
    """Solved plans saved as JSON lines reload bit-identically without re-solving
    (the reloaded solve_us is the saved one), and foreign lines are skipped."""
    import json
    from paper_2412_07752_b200 import abi
    abi.plan_cache_clear()
    before = [abi.plan(*s) for s in CACHE_SHAPES]
    path = tmp_path / "plans.jsonl"
    abi.plan_cache_save(path)
    lines = path.read_text().splitlines()
    assert len(lines) == len(CACHE_SHAPES)
    for ln in lines:
        j = json.loads(ln)
        assert j["schema_version"] == 1 and j["version"] == abi.version() and j["sm_count"] > 0
    # a line from another build, a truncated line and noise are ignored
    other = json.loads(lines[0])
    other["version"] = "flashrnn-b200 0.0.0 (other build)"
    other["batch"] = 999
    path.write_text("\n".join(lines + [json.dumps(other), lines[1][:40], "not json"]) + "\n")
    abi.plan_cache_clear()
    assert abi.plan_cache_load(path) == len(CACHE_SHAPES)
    after = [abi.plan(*s) for s in CACHE_SHAPES]
    assert after == before  # including solve_us: served from the cache, not re-solved
    with pytest.raises(abi.FrnnError):
        abi.plan_cache_load(tmp_path / "missing.jsonl")


def test_plan_cache_env_persists_across_processes(tmp_path):
    """FRNN_PLAN_CACHE=<file>: the first process solves and appends, the second
    starts from the file and reports the first one's solve time."""
    import json
    import os
    import subprocess
    import sys
    path = tmp_path / "env_plans.jsonl"
    code = ("import json, sys; sys.path.insert(0, %r); from paper_2412_07752_b200 import abi; "
            "print(json.dumps(abi.plan('slstm', 1024, 16, 1, 768, 'bf16', 'backward')))"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    env = dict(os.environ, FRNN_PLAN_CACHE=str(path))
    runs = [json.loads(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                                      check=True).stdout.strip().splitlines()[-1]) for _ in range(2)]
    assert runs[0] == runs[1]
    assert len(path.read_text().splitlines()) == 1  # the second process did not solve again
