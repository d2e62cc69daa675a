"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerances (stated here and in DESIGN.md section 6):
  * fp32 mode: normwise relative error ||gpu - oracle_f64|| / ||oracle_f64|| <= 1e-5
    per output tensor (the reference's own float engine sits at 1e-7..1e-6 on
    config 1; elementwise rel is not used because ~0 entries make it ill-posed).
  * bf16 mode: inputs rounded to bf16 RNE, oracle = the f64 engine on the rounded
    inputs; normwise relative error <= 2e-2 per tensor:
      - forward: states, gates vs the oracle forward on the same inputs;
      - backward: dx, dbias, dR, ds0 vs the oracle backward on the same inputs,
        which for rnnkit's backward (engine.hpp:222) include the trace -- so the
        oracle backward is fed the trace the GPU forward produced;
      - end to end (oracle trace): same 2e-2 for Elman/LSTM/GRU.  The sLSTM
        gradient is discontinuous at the stabilizer tie a == i (the max branch,
        cell.hpp:153), so bf16-level differences in the trace flip a handful of
        near-tie elements and move the normwise gradient error by what the bf16
        format alone costs.  That cost is measured per case as the CONTROL
        (conftest.trace_control): the oracle's own backward on its f64 trace
        perturbed to the GPU trace's measured distance and rounded to bf16, vs
        on the f64 trace, max over 8 realizations (the plain-rounding control
        is pinned on the CPU by tests/test_oracle.py::test_bf16_trace_control);
        sLSTM end to end is bounded by 2e-2 + max(control, sensitivity) per
        gradient, where sensitivity = the oracle backward on the GPU's own
        (forward-checked) bf16 trace vs on the f64 trace: at small T the random
        realizations need not flip the same near-tie elements the GPU trace flips.
    Full-length (T=1024) versions of these checks: tests/test_full_length_parity.py.
"""
import numpy as np
import pytest

from conftest import normwise, trace_control

pytestmark = pytest.mark.gpu

VARIANTS = ["elman", "lstm", "gru", "slstm"]
FP32_TOL = 1e-5
BF16_TOL = 2e-2
GRADS = ("dx", "dbias", "dR", "ds0")


@pytest.fixture(scope="module")
def eng():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2412_07752_b200 import FlashRNN
    return FlashRNN()


def _dev(a, dt):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dt).contiguous()


def _np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def run_gpu(eng, v, inp, bf16, clip="off", mag=0.0, dh=None, algo="auto"):
    import torch
    dt = torch.bfloat16 if bf16 else torch.float32
    R, b, x, s0, dsf = (_dev(inp[k], dt) for k in ("R", "bias", "x", "s0", "dsf"))
    st, ga = eng.forward(v, R, b, x, s0, algo=algo)
    g = eng.backward(v, R, b, st, ga, dsf, None if dh is None else _dev(dh, dt), clip, mag, algo=algo)
    torch.cuda.synchronize()
    out = {k: _np(t) for k, t in g.items()}
    out["states"], out["gates"] = _np(st), _np(ga)
    return out


def run_oracle(orc, v, inp, bf16, clip="off", mag=0.0, dh=None):
    if bf16:
        inp = {k: orc.round_bf16(a) for k, a in inp.items()}
        dh = orc.round_bf16(dh) if dh is not None else None
    st, ga = orc.forward(v, inp["R"], inp["bias"], inp["x"], inp["s0"])
    g = orc.backward(v, inp["R"], st, ga, inp["dsf"], clip, mag, dh)
    g["states"], g["gates"] = st, ga
    return g


def assert_close(gpu, ora, tol, keys=("states", "gates", "dx", "dbias", "dR", "ds0")):
    errs = {k: normwise(gpu[k], ora[k]) for k in keys}
    bad = {k: e for k, e in errs.items() if not e <= tol}
    assert not bad, f"normwise errors above {tol}: {bad} (all: {errs})"
    return errs


def check_bf16(eng, orc, v, inp, clip="off", mag=0.0, dh=None, algo="auto"):
    gpu = run_gpu(eng, v, inp, True, clip, mag, dh, algo)
    ora = run_oracle(orc, v, inp, True, clip, mag, dh)
    fwd = assert_close(gpu, ora, BF16_TOL, ("states", "gates"))
    r = {k: orc.round_bf16(inp[k]) for k in ("R", "dsf")}
    cond = orc.backward(v, r["R"], gpu["states"], gpu["gates"], r["dsf"], clip, mag,
                        orc.round_bf16(dh) if dh is not None else None)
    bwd = assert_close(gpu, cond, BF16_TOL, GRADS)
    e2e = {k: normwise(gpu[k], ora[k]) for k in GRADS}
    if v == "slstm":
        ctl, _ = trace_control(orc, v, r["R"], ora["states"], ora["gates"], r["dsf"],
                               fwd["states"], 8, clip, mag,
                               orc.round_bf16(dh) if dh is not None else None)
        # the oracle's response to the exact bf16 trace the GPU produced (checked
        # above): at small T the random realizations may flip other near-tie
        # elements than the GPU trace does, so the bound takes the larger of the two
        sens = {k: normwise(cond[k], ora[k]) for k in GRADS}
        bad = {k: (e2e[k], ctl[k], sens[k]) for k in GRADS
               if not e2e[k] <= BF16_TOL + max(ctl[k], sens[k])}
        assert not bad, ("sLSTM end to end above max(control, trace sensitivity) + 2e-2", bad)
    else:
        assert max(e2e.values()) <= BF16_TOL, e2e
    print(v, "fwd", fwd, "bwd(same trace)", bwd, "e2e", e2e)
    return fwd, bwd, e2e


# ------------------------------------------------------------- fp32 mode ----
def test_config1_lstm_fp32(eng, orc):
    """BASELINE config 1: LSTM fp32, 1 head, D=64, B=8, T=64."""
    inp = orc.generate("lstm", 64, 8, 1, 64, seed=0)
    errs = assert_close(run_gpu(eng, "lstm", inp, False), run_oracle(orc, "lstm", inp, False), FP32_TOL)
    print("config1 normwise:", errs)


def test_config1_against_reference_engine(eng, ref):
    """Same inputs through the unmodified reference (oracle/_ref) in double."""
    inp = ref.generate("lstm", 64, 8, 1, 64, seed=0)
    st, ga = ref.forward("lstm", inp["R"], inp["bias"], inp["x"], inp["s0"])
    g = ref.backward("lstm", inp["R"], inp["bias"], inp["x"], inp["s0"], st, ga, inp["dsf"])
    g["states"], g["gates"] = st, ga
    assert_close(run_gpu(eng, "lstm", inp, False), g, FP32_TOL)


@pytest.mark.parametrize("v", VARIANTS)
@pytest.mark.parametrize("clip,mag", [("off", 0.0), ("value", 0.05), ("zero", 0.0)])
def test_fp32_variants(eng, orc, v, clip, mag):
    inp = orc.generate(v, 12, 5, 2, 24, seed=3)
    assert_close(run_gpu(eng, v, inp, False, clip, mag), run_oracle(orc, v, inp, False, clip, mag), FP32_TOL)


@pytest.mark.parametrize("v", VARIANTS)
def test_fp32_step_gradients(eng, orc, v):
    inp = orc.generate(v, 9, 11, 1, 40, seed=4)
    dh = np.random.RandomState(1).randn(9, 11, 40)
    assert_close(run_gpu(eng, v, inp, False, dh=dh), run_oracle(orc, v, inp, False, dh=dh), FP32_TOL)


def test_fp32_golden(eng):
    """Golden vectors produced by the reference's float engine."""
    import os
    for v in VARIANTS:
        g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", f"{v}_small.npz")))
        out = run_gpu(eng, v, g, False)
        for k in ("states", "gates"):
            assert normwise(out[k], g[f"f32_{k}"]) <= FP32_TOL, (v, k)
        for k in ("dx", "dbias", "dR", "ds0"):
            assert normwise(out[k], g[f"f32_off_{k}"]) <= FP32_TOL, (v, k)


# ------------------------------------------------------------- bf16 mode ----
@pytest.mark.parametrize("v", VARIANTS)
@pytest.mark.parametrize("clip,mag", [("off", 0.0), ("value", 0.05), ("zero", 0.0)])
def test_fp32_beyond_shared_memory(eng, orc, v, clip, mag):
    """fp32 mode with R too large for the SIMT kernels' shared memory (DH=128,
    two heads, ragged batch): the streamed FFMA path (alt_fp32.cu), rel 1e-5."""
    inp = orc.generate(v, 6, 19, 2, 128, seed=12)
    dh = np.random.RandomState(4).randn(6, 19, 256)
    if v != "elman":  # a single-gate R still fits the SIMT kernels at DH=128
        assert eng.plan(v, 6, 19, 2, 128, "f32", "backward")["algo"] == 2
    gpu = run_gpu(eng, v, inp, False, clip, mag, dh, algo="alternating")
    assert_close(gpu, run_oracle(orc, v, inp, False, clip, mag, dh), FP32_TOL)


@pytest.mark.parametrize("v", ["lstm", "slstm"])
def test_fp32_h768(eng, orc, v):
    """fp32 mode at the headline shape (B=16, H=768, NH=1), reduced T."""
    inp = orc.generate(v, 4, 16, 1, 768, seed=13)
    assert_close(run_gpu(eng, v, inp, False), run_oracle(orc, v, inp, False), FP32_TOL)


@pytest.mark.parametrize("v", VARIANTS)
def test_bf16_fused_h768(eng, orc, v):
    """Configs 2/4 shape (H=768, NH=1, B=16) at reduced T (oracle cost)."""
    inp = orc.generate(v, 24, 16, 1, 768, seed=0)
    check_bf16(eng, orc, v, inp)


@pytest.mark.parametrize("v", ["slstm", "gru"])
def test_bf16_cluster_three_batch_tiles(eng, orc, v):
    """H=768 with B=40: three 16-row clusters per head (the last ragged) on the
    cluster kernels' paired TMEM/SMEM column blocks."""
    inp = orc.generate(v, 6, 40, 1, 768, seed=12)
    assert eng.plan(v, 6, 40, 1, 768, "bf16", "backward")["cluster"] == 16
    check_bf16(eng, orc, v, inp)


@pytest.mark.parametrize("v,NH,DH,B", [("slstm", 1, 640, 24), ("slstm", 1, 896, 20), ("lstm", 2, 384, 24),
                                       ("elman", 1, 512, 16), ("gru", 1, 512, 16)])
def test_bf16_other_head_dims(eng, orc, v, NH, DH, B):
    """Head dims whose tilings differ from the headline: DH=640 (UPC=40, five
    TMEM blocks, no SMEM block), DH=896 (no single-cluster tiling: two-cluster
    forward + alternating backward), two heads of 384, Elman 512."""
    inp = orc.generate(v, 6, B, NH, DH, seed=13)
    check_bf16(eng, orc, v, inp)


@pytest.mark.parametrize("v,NH,DH,B,ncl", [("lstm", 1, 1024, 16, 2), ("slstm", 1, 1024, 20, 2),
                                           ("gru", 1, 1152, 16, 3), ("elman", 1, 1024, 8, 2),
                                           ("slstm", 2, 896, 16, 2), ("lstm", 1, 1408, 16, 4),
                                           ("gru", 1, 1536, 16, 6)])
def test_bf16_multicluster(eng, orc, v, NH, DH, B, ncl):
    """R-resident forward beyond one cluster (fused_cluster.cu, NCL > 1): the
    head's units over NCL clusters, h slices of the other clusters imported
    through L2 behind release counters; DH > 960 also splits each CTA's R rows
    along K between TMEM and an SMEM M=128 tile.  B=20: two batch tiles; NH=2:
    two heads.  Backward: multi-cluster for the 4-gate tilings with an issue
    instance (DH 896/1024/1152), else alternating."""
    pf = eng.plan(v, 6, B, NH, DH, "bf16", "forward")
    assert pf["algo"] == 1 and pf["ctas_per_group"] == ncl * pf["cluster"], pf
    inp = orc.generate(v, 6, B, NH, DH, seed=21)
    check_bf16(eng, orc, v, inp)


@pytest.mark.parametrize("v,NH,DH,B", [("lstm", 1, 1024, 16), ("slstm", 1, 1024, 20), ("gru", 1, 1152, 16),
                                       ("slstm", 2, 896, 24), ("lstm", 1, 960, 16), ("gru", 1, 832, 8)])
def test_bf16_multicluster_backward(eng, orc, monkeypatch, v, NH, DH, B):
    """The multi-cluster backward (FRNN_MC_BWD=1: for any tiling): R^T.dg
    partials for owners in other clusters stored to L2 and pulled by TMA after
    their sources' release counters, summed after the own cluster's DSMEM
    partials in a fixed order.  (Shapes not planned by any other test: the
    plan cache is per shape.)"""
    monkeypatch.setenv("FRNN_MC_BWD", "1")
    pb = eng.plan(v, 7, B, NH, DH, "bf16", "backward")
    assert pb["algo"] == 1 and pb["ctas_per_group"] > pb["cluster"], pb
    inp = orc.generate(v, 7, B, NH, DH, seed=22)
    check_bf16(eng, orc, v, inp)


@pytest.mark.parametrize("v,clip,mag", [("slstm", "value", 0.05), ("lstm", "zero", 0.0), ("gru", "off", 0.0)])
def test_bf16_multicluster_clip_ragged_step_grads(eng, orc, v, clip, mag):
    """Multi-cluster forward + backward (H=1024, two clusters) with gradient
    clipping (the remote partials are summed before the clip), a ragged second
    batch tile (B=21) and per-step hidden gradients."""
    T, B, DH = 8, 21, 1024
    assert eng.plan(v, T, B, 1, DH, "bf16", "backward")["ctas_per_group"] == 32
    inp = orc.generate(v, T, B, 1, DH, seed=23)
    dh = 0.5 * np.random.RandomState(3).randn(T, B, DH)
    check_bf16(eng, orc, v, inp, clip, mag, dh=dh)


@pytest.mark.parametrize("T", [0, 1, 2])
def test_multicluster_short_sequences(eng, orc, T):
    """Multi-cluster kernels (H=1024, two clusters per pass) at T = 0 / 1 / 2:
    no step, a single step (no h exchange at all), one exchange."""
    inp = orc.generate("lstm", T, 16, 1, 1024, seed=41)
    assert eng.plan("lstm", T, 16, 1, 1024, "bf16", "forward")["ctas_per_group"] == 32
    gpu = run_gpu(eng, "lstm", inp, True)
    ora = run_oracle(orc, "lstm", inp, True)
    keys = ("states", "dbias", "dR", "ds0") + (("gates", "dx") if T else ())
    assert_close(gpu, ora, BF16_TOL, keys)


def test_multicluster_falls_back_when_not_coresident(eng, orc):
    """B=256 at H=1024 needs 16 batch tiles x 2 clusters of 16 CTAs: more
    clusters than can be resident at once, so the planner must not pick the
    multi-cluster kernels (they spin on each other); the fallback is correct."""
    pf = eng.plan("lstm", 2, 256, 1, 1024, "bf16", "forward")
    assert not (pf["algo"] == 1 and pf["ctas_per_group"] > pf["cluster"] > 0), pf
    inp = orc.generate("lstm", 2, 256, 1, 1024, seed=42)
    check_bf16(eng, orc, "lstm", inp)


@pytest.mark.parametrize("NH,DH", [(1, 768), (1, 512), (2, 96)])
def test_bf16_gru_compact_k(eng, orc, monkeypatch, NH, DH):
    """GRU backward with the n gate's (zero) R rows dropped from the R^T.dg K
    dimension (FRNN_GRU_COMPACT=1, cell.hpp:43): same results as the padded layout."""
    monkeypatch.setenv("FRNN_GRU_COMPACT", "1")
    inp = orc.generate("gru", 12, 16, NH, DH, seed=5)
    check_bf16(eng, orc, "gru", inp)


@pytest.mark.parametrize("B", [5, 24, 40, 48, 96, 130])
def test_bf16_dr_gemm_any_batch(eng, orc, B):
    """dR / db through the tcgen05 dR GEMM (dr_gemm.cu) at batch sizes that do
    not divide its 64-deep K tile (engine.hpp:321-334 summed over t and b):
    whole steps per tile for B <= 64 (zero-padded K rows), 64-row batch chunks
    for B > 64.  Same-trace check against the oracle backward."""
    v, T, NH, DH = "lstm", 7, 1, 128
    inp = {k: orc.round_bf16(a) for k, a in orc.generate(v, T, B, NH, DH, seed=B).items()}
    gpu = run_gpu(eng, v, inp, True)
    cond = orc.backward(v, inp["R"], gpu["states"], gpu["gates"], inp["dsf"])
    errs = assert_close(gpu, cond, BF16_TOL, ("dR", "dbias", "dx"))
    print("B", B, errs)


@pytest.mark.parametrize("pbf16", ["0", "1"])
def test_bf16_partial_exchange_modes(eng, orc, monkeypatch, pbf16):
    """The backward's R^T.dg partials as fp32 (FRNN_PBF16=0) or bf16 pairs (the
    default for 4-gate cells): both within the bf16 tolerance."""
    monkeypatch.setenv("FRNN_PBF16", pbf16)
    inp = orc.generate("slstm", 12, 16, 1, 768, seed=14)
    check_bf16(eng, orc, "slstm", inp)


@pytest.mark.parametrize("NH,DH", [(4, 192), (12, 64)])
def test_bf16_lstm_heads(eng, orc, NH, DH):
    """Config 3: head-wise block-diagonal R."""
    inp = orc.generate("lstm", 48, 16, NH, DH, seed=1)
    check_bf16(eng, orc, "lstm", inp)


@pytest.mark.parametrize("v", VARIANTS)
@pytest.mark.parametrize("clip,mag", [("value", 0.05), ("zero", 0.0)])
def test_bf16_clip(eng, orc, v, clip, mag):
    inp = orc.generate(v, 16, 16, 2, 64, seed=2)
    check_bf16(eng, orc, v, inp, clip, mag)


@pytest.mark.parametrize("v", VARIANTS)
def test_bf16_ragged_batch_and_step_grads(eng, orc, v):
    """B=21 -> two batch tiles, the second ragged; per-step hidden gradients."""
    inp = orc.generate(v, 10, 21, 2, 48, seed=5)
    dh = np.random.RandomState(2).randn(10, 21, 96)
    check_bf16(eng, orc, v, inp, dh=dh)


@pytest.mark.parametrize("T", [0, 1])
def test_edge_seq_len(eng, orc, T):
    for v in VARIANTS:
        for bf16 in (False, True):
            inp = orc.generate(v, T, 3, 1, 32, seed=6)
            gpu = run_gpu(eng, v, inp, bf16)
            ora = run_oracle(orc, v, inp, bf16)
            tol = BF16_TOL if bf16 else FP32_TOL
            keys = ("states", "dbias", "dR", "ds0") + (("gates", "dx") if T else ())
            assert_close(gpu, ora, tol, keys)


def test_bf16_golden(eng, orc):
    """Golden (reference) inputs through the bf16 path vs f64 on rounded inputs."""
    import os
    for v in VARIANTS:
        g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", f"{v}_small.npz")))
        check_bf16(eng, orc, v, {k: g[k] for k in ("R", "bias", "x", "s0", "dsf")})


# ------------------------------------------- alternating path (K4/K5) ----
@pytest.mark.parametrize("v", VARIANTS)
def test_alternating_variants(eng, orc, v):
    """Per-step streamed-R kernels (forced), two heads, ragged batch tile."""
    inp = orc.generate(v, 12, 21, 2, 128, seed=3)
    check_bf16(eng, orc, v, inp, algo="alternating")


@pytest.mark.parametrize("v", VARIANTS)
@pytest.mark.parametrize("clip,mag", [("value", 0.05), ("zero", 0.0)])
def test_alternating_clip_and_step_grads(eng, orc, v, clip, mag):
    inp = orc.generate(v, 8, 16, 1, 192, seed=4)
    dh = np.random.RandomState(3).randn(8, 16, 192)
    check_bf16(eng, orc, v, inp, clip, mag, dh=dh, algo="alternating")


def test_alternating_two_batch_tiles(eng, orc):
    """B=160: batch tiles of 128 (the second ragged), per-tile db partials."""
    inp = orc.generate("lstm", 6, 160, 1, 128, seed=7)
    check_bf16(eng, orc, "lstm", inp, algo="alternating")


@pytest.mark.parametrize("v,NH,DH", [("lstm", 3, 20), ("gru", 2, 36), ("slstm", 1, 12), ("elman", 1, 1000)])
def test_bf16_untileable_head_dims(eng, orc, v, NH, DH):
    """bf16 head dims no tensor-core kernel tiles (not a multiple of 8, or past
    the fused limits and not a multiple of 64): FFMA step kernels, bf16 storage."""
    T = 4 if DH > 256 else 10
    inp = orc.generate(v, T, 19, NH, DH, seed=11)
    dh = np.random.RandomState(5).randn(T, 19, NH * DH)
    check_bf16(eng, orc, v, inp, dh=dh)


def test_alternating_matches_fused(eng, orc):
    """Same inputs through the cluster-resident and the alternating kernels."""
    inp = orc.generate("slstm", 16, 16, 1, 768, seed=8)
    a = run_gpu(eng, "slstm", inp, True, algo="fused")
    b = run_gpu(eng, "slstm", inp, True, algo="alternating")
    assert_close(b, a, BF16_TOL, ("states", "gates"))


def test_config5_slstm_h3072(eng, orc):
    """BASELINE config 5 shape: sLSTM H=3072, B=64, NH=1 (R = 75.5 MB, beyond
    on-chip capacity -> the planner picks the alternating path); T=3 (oracle cost)."""
    p = eng.plan("slstm", 3, 64, 1, 3072, "bf16", "backward")
    assert p["algo"] == 2, p
    inp = orc.generate("slstm", 3, 64, 1, 3072, seed=0)
    check_bf16(eng, orc, "slstm", inp)


def test_config5_full_size_properties(eng, orc):
    """sLSTM H=3072, B=64, T=1024: deterministic, finite, causal prefix parity."""
    import torch
    T, B, DH, NS, NG = 1024, 64, 3072, 4, 4
    g = torch.Generator(device="cuda").manual_seed(0)
    R = (torch.randn(1, NG, DH, DH, device="cuda", generator=g) / DH ** 0.5).bfloat16()
    b = (0.1 * torch.randn(NG, DH, device="cuda", generator=g)).bfloat16()
    x = torch.randn(T, B, NG, DH, device="cuda", generator=g).bfloat16()
    s0 = 0.5 * torch.randn(NS, B, DH, device="cuda", generator=g)
    s0[2] = 1 + 0.1 * s0[2].abs()
    s0[3] = 0
    s0 = s0.bfloat16()
    dsf = torch.randn(NS, B, DH, device="cuda", generator=g).bfloat16()
    st1, ga1 = eng.forward("slstm", R, b, x, s0)
    gr1 = eng.backward("slstm", R, b, st1, ga1, dsf)
    st2, ga2 = eng.forward("slstm", R, b, x, s0)
    gr2 = eng.backward("slstm", R, b, st2, ga2, dsf)
    torch.cuda.synchronize()
    assert torch.equal(st1, st2) and torch.equal(ga1, ga2)
    for k in gr1:
        assert torch.equal(gr1[k], gr2[k]), k
        assert torch.isfinite(gr1[k].float()).all(), k
    assert torch.isfinite(st1.float()).all()
    P = 2
    ost, oga = orc.forward("slstm", _np(R), _np(b), _np(x[:P]), _np(s0))
    assert normwise(_np(st1[: P + 1]), ost) <= BF16_TOL
    assert normwise(_np(ga1[:P]), oga) <= BF16_TOL


# ---------------------------------------------- full-size property tests ----
@pytest.mark.parametrize("v", ["slstm", "lstm"])
def test_full_size_prefix_and_determinism(eng, orc, v):
    """B=16, T=1024, H=768: the forward is causal, so states[0..32] of the full
    run must match an oracle T=32 run on the same prefix; two runs must be
    bit-identical; everything finite."""
    import torch
    T, B, DH = 1024, 16, 768
    g = torch.Generator(device="cuda").manual_seed(0)
    NS, NG = (4, 4) if v == "slstm" else (2, 4)
    R = (torch.randn(1, NG, DH, DH, device="cuda", generator=g) / DH ** 0.5).bfloat16()
    b = (0.1 * torch.randn(NG, DH, device="cuda", generator=g)).bfloat16()
    x = torch.randn(T, B, NG, DH, device="cuda", generator=g).bfloat16()
    s0 = (0.5 * torch.randn(NS, B, DH, device="cuda", generator=g))
    if v == "slstm":
        s0[2] = 1 + 0.1 * s0[2].abs()
        s0[3] = 0
    s0 = s0.bfloat16()
    dsf = torch.randn(NS, B, DH, device="cuda", generator=g).bfloat16()
    st1, ga1 = eng.forward(v, R, b, x, s0)
    gr1 = eng.backward(v, R, b, st1, ga1, dsf)
    st2, ga2 = eng.forward(v, R, b, x, s0)
    gr2 = eng.backward(v, R, b, st2, ga2, dsf)
    torch.cuda.synchronize()
    assert torch.equal(st1, st2) and torch.equal(ga1, ga2)
    for k in gr1:
        assert torch.equal(gr1[k], gr2[k]), k
        assert torch.isfinite(gr1[k].float()).all(), k
    assert torch.isfinite(st1.float()).all()
    P = 32
    ost, oga = orc.forward(v, _np(R), _np(b), _np(x[:P]), _np(s0))
    assert normwise(_np(st1[: P + 1]), ost) <= BF16_TOL
    assert normwise(_np(ga1[:P]), oga) <= BF16_TOL


def test_backward_linearity_full_size(eng):
    """BPTT is linear in the incoming gradients: bwd(2a + b) = 2 bwd(a) + bwd(b)."""
    import torch
    T, B, DH, NH = 1024, 16, 192, 4
    g = torch.Generator(device="cuda").manual_seed(1)
    R = (torch.randn(NH, 4, DH, DH, device="cuda", generator=g) / DH ** 0.5).bfloat16()
    bias = (0.1 * torch.randn(4, NH * DH, device="cuda", generator=g)).bfloat16()
    x = torch.randn(T, B, 4, NH * DH, device="cuda", generator=g).bfloat16()
    s0 = (0.5 * torch.randn(2, B, NH * DH, device="cuda", generator=g)).bfloat16()
    st, ga = eng.forward("lstm", R, bias, x, s0)
    da = torch.randn(2, B, NH * DH, device="cuda", generator=g).bfloat16()
    db = torch.randn(2, B, NH * DH, device="cuda", generator=g).bfloat16()
    ga_ = eng.backward("lstm", R, bias, st, ga, da)
    gb_ = eng.backward("lstm", R, bias, st, ga, db)
    gc_ = eng.backward("lstm", R, bias, st, ga, (2 * da.float() + db.float()).bfloat16())
    for k in ("dR", "dbias"):  # ds0 after 1024 steps is at the bf16 noise floor
        lhs = gc_[k].double()
        rhs = 2 * ga_[k].double() + gb_[k].double()
        assert ((lhs - rhs).norm() / rhs.norm()).item() < 3e-2, k


def test_nonfinite_rejected(eng):
    import torch
    from paper_2412_07752_b200 import FrnnError
    R = torch.zeros(1, 4, 16, 16, device="cuda")
    b = torch.zeros(4, 16, device="cuda")
    x = torch.zeros(3, 2, 4, 16, device="cuda")
    x[1, 0, 2, 3] = float("nan")
    s0 = torch.zeros(2, 2, 16, device="cuda")
    with pytest.raises(FrnnError) as ei:
        eng.forward("lstm", R, b, x, s0, check_finite=True)
    assert ei.value.status == "ENONFINITE"
