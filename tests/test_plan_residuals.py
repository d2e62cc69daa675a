"""Plan verification (the tiling solver): every plan the planner
returns passes its residual check -- the B200 counterpart of
rnnkit::plan::plan_residuals (planner.cpp:349-402): the derived geometry
(shared memory, TMEM columns, threads, grid, workspace) recomputed from the
plan's choices equals the plan's values and every family constraint holds --
and a corrupted plan is rejected.  The per-step traffic model (the counterpart
of hbm_traffic_per_step, planner.cpp:233-243) is checked against its closed
form.  CPU only (no device: the device limits are B200's)."""
import ctypes as C
import json

import pytest

from paper_2412_07752_b200.abi import ALGO, DTYPE, PASS, Options, Shape, cell_spec, load

VARIANTS = ["elman", "lstm", "gru", "slstm"]


def _lib():
    L = load()
    L.frnn_plan_check.argtypes = [C.c_void_p, Shape, C.c_int32, C.c_int32, C.c_void_p, C.c_char_p, C.c_size_t]
    L.frnn_debug_plan_fields.argtypes = [C.c_void_p, Shape, C.c_int32, C.c_int32, C.c_void_p,
                                         C.POINTER(C.c_int64)]
    L.frnn_debug_plan_residuals.argtypes = [C.c_void_p, Shape, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                            C.c_char_p, C.c_size_t]
    L.frnn_plan_json.argtypes = [C.c_void_p, Shape, C.c_int32, C.c_int32, C.c_void_p, C.c_char_p, C.c_size_t]
    return L


def check(L, v, T, B, NH, DH, dt, ps, algo="auto"):
    buf = C.create_string_buffer(8192)
    o = Options(0, ALGO[algo])
    rc = L.frnn_plan_check(C.byref(cell_spec(v)), Shape(T, B, NH, DH), DTYPE[dt], PASS[ps], C.byref(o), buf, 8192)
    return rc, json.loads(buf.value.decode() or "null")


@pytest.mark.parametrize("v", VARIANTS)
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_every_plan_has_zero_residuals(v, dt):
    L = _lib()
    n = 0
    for DH in (16, 48, 64, 96, 192, 256, 384, 512, 640, 768, 896, 1024, 1152, 1408, 1536, 3072):
        for B, NH in ((8, 1), (16, 1), (40, 2), (64, 1)):
            for ps in ("forward", "backward"):
                rc, res = check(L, v, 64, B, NH, DH, dt, ps)
                assert rc == 0 and res == [], (v, dt, DH, B, NH, ps, rc, res)
                n += 1
    assert n == 16 * 4 * 2


def _fields(L, v, DH, B, ps, algo="auto"):
    f = (C.c_int64 * 16)()
    o = Options(0, ALGO[algo])
    assert L.frnn_debug_plan_fields(C.byref(cell_spec(v)), Shape(64, B, 1, DH), DTYPE["bf16"], PASS[ps],
                                    C.byref(o), f) == 0
    return f


def _residuals(L, v, DH, B, ps, f):
    buf = C.create_string_buffer(8192)
    rc = L.frnn_debug_plan_residuals(C.byref(cell_spec(v)), Shape(64, B, 1, DH), DTYPE["bf16"], PASS[ps], f,
                                     buf, 8192)
    return rc, json.loads(buf.value.decode())


@pytest.mark.parametrize("field,delta,needle", [(8, 16, "shared memory"), (6, 1, "grid"), (3, 8, "units per CTA"),
                                                (9, 256, "TMEM"), (15, 256, "workspace"), (7, 32, "threads")])
@pytest.mark.parametrize("v,DH,B,ps", [("slstm", 768, 16, "forward"), ("lstm", 768, 16, "backward"),
                                       ("lstm", 1024, 16, "forward")])
def test_corrupted_cluster_plans_are_rejected(v, DH, B, ps, field, delta, needle):
    L = _lib()
    f = _fields(L, v, DH, B, ps)
    assert f[0] == 1 and f[11] > 0, list(f)  # cluster-resident (one or several clusters)
    assert _residuals(L, v, DH, B, ps, f) == (0, [])
    f[field] += delta
    rc, res = _residuals(L, v, DH, B, ps, f)
    assert rc == 4 and any(needle in r for r in res), (field, res)


def test_corrupted_alternating_plan_is_rejected():
    L = _lib()
    f = _fields(L, "slstm", 3072, 64, "backward")
    assert f[0] == 2 and _residuals(L, "slstm", 3072, 64, "backward", f) == (0, [])
    f[13] += 2  # ring stages: shared memory / region no longer match
    rc, res = _residuals(L, "slstm", 3072, 64, "backward", f)
    assert rc == 4 and res, res


def _json(L, v, T, B, NH, DH, ps):
    buf = C.create_string_buffer(4096)
    o = Options(0, ALGO["auto"])
    assert L.frnn_plan_json(C.byref(cell_spec(v)), Shape(T, B, NH, DH), DTYPE["bf16"], PASS[ps], C.byref(o), buf,
                            4096) == 0
    return json.loads(buf.value.decode())


def test_traffic_model_closed_form():
    L = _lib()
    B, D = 16, 768
    # headline forward (sLSTM: 4 gates, 4 states, every gate input-wired), cluster of 16
    j = _json(L, "slstm", 1024, B, 1, D, "forward")
    t = j["traffic_per_step_bytes"]
    assert t["io"] == B * (4 + 4 + 4) * D * 2 and t["r_stream"] == 0
    assert t["exchange_l2"] == B * D * 2 and t["exchange_onchip"] == B * D * 2 * 16 and j["residuals"] == 0
    # headline backward: trace in (4 states + 4 gates), dx out; bf16-pair partials through DSMEM
    t = _json(L, "slstm", 1024, B, 1, D, "backward")["traffic_per_step_bytes"]
    assert t["io"] == B * (4 + 4 + 4) * D * 2 and t["exchange_onchip"] == B * D * 2 * 16 and t["exchange_l2"] == 0
    # config 5 (alternating): R re-read from L2 every step, fp32 carries
    t = _json(L, "slstm", 1024, 64, 1, 3072, "forward")["traffic_per_step_bytes"]
    assert t["r_stream"] == 4 * 3072 * 3072 * 2
    assert t["io"] == 64 * 12 * 3072 * 2 + 2 * 4 * 64 * 3072 * 4


@pytest.mark.gpu
@pytest.mark.parametrize("v", VARIANTS)
def test_every_plan_has_zero_residuals_on_device(v):
    """The same sweep on a B200: the device-queried limits, the co-residency of
    multi-cluster groups (cudaOccupancyMaxActiveClusters) and the compiled
    kernels' registers x threads enter the check."""
    import torch
    assert torch.cuda.is_available()
    L = _lib()
    for DH in (64, 192, 512, 768, 896, 1024, 1152, 1536, 1792, 3072):
        for B, NH in ((16, 1), (40, 2), (64, 1)):
            for ps in ("forward", "backward"):
                rc, res = check(L, v, 64, B, NH, DH, "bf16", ps)
                assert rc == 0 and res == [], (v, DH, B, NH, ps, rc, res)
