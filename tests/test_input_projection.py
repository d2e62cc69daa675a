"""The input projection before the recurrence (frnn_input_projection, SURVEY 8f
row 1): x[T][B][NG*D] = u[T][B][Din] . W^T on tcgen05 (csrc/wx_gemm.cu).

Oracle: float64 matmul of the same bf16-rounded inputs; the result is rounded
to bf16 once, so the normwise error bound is a few bf16 ulps (tolerance 4e-3
normwise, stated here)."""
import ctypes as C

import numpy as np
import pytest

from paper_2412_07752_b200.abi import FrnnError, load

TOL = 4e-3


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def test_abi_validation_without_gpu():
    L = load()
    L.frnn_input_projection.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_void_p]
    buf = C.create_string_buffer(64)
    p = C.cast(buf, C.c_void_p)
    assert L.frnn_input_projection(None, p, p, 4, 8, 8, 1, None) == 6          # EINVAL_ARG
    assert L.frnn_input_projection(p, p, p, 0, 8, 8, 1, None) == 1             # EINVAL_SHAPE
    assert L.frnn_input_projection(p, p, p, 4, 8, 12, 1, None) == 1            # in_features % 8
    assert L.frnn_input_projection(p, p, p, 4, 8, 8, 0, None) == 3             # fp32: EUNSUPPORTED


@pytest.mark.gpu
@pytest.mark.parametrize("T,B,Din,NG,D", [(5, 3, 96, 4, 80), (7, 16, 64, 1, 256), (3, 21, 200, 4, 48),
                                          (4, 5, 64, 1, 36), (9, 40, 136, 3, 200), (300, 9, 64, 4, 72)])
def test_ragged_shapes(T, B, Din, NG, D):
    """Token and gate tails inside a 256x256 pair tile, a K tail (Din=200, 136),
    out_features % 8 != 0 (the single-CTA kernel) and more tiles than pairs."""
    import torch
    from paper_2412_07752_b200 import FlashRNN
    g = torch.Generator(device="cuda").manual_seed(T * 100 + Din)
    u = torch.randn(T, B, Din, device="cuda", generator=g).bfloat16()
    W = (torch.randn(NG * D, Din, device="cuda", generator=g) / Din ** 0.5).bfloat16()
    x = FlashRNN().input_projection(W, u)
    torch.cuda.synchronize()
    ref = _np(u).reshape(-1, Din) @ _np(W).T
    got = _np(x).reshape(-1, NG * D)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= TOL, err


@pytest.mark.gpu
def test_headline_shape_and_throughput():
    """T=1024, B=16, Din=768 -> NG*D = 4*768 (configs 2-4): sampled rows vs the
    oracle, plus the achieved TFLOP/s (printed)."""
    import torch
    from paper_2412_07752_b200 import FlashRNN
    T, B, Din, N = 1024, 16, 768, 3072
    g = torch.Generator(device="cuda").manual_seed(7)
    u = torch.randn(T, B, Din, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, Din, device="cuda", generator=g) / Din ** 0.5).bfloat16()
    eng = FlashRNN()
    x = eng.input_projection(W, u)
    rows = np.random.RandomState(0).choice(T * B, 96, replace=False)
    ref = _np(u).reshape(-1, Din)[rows] @ _np(W).T
    got = _np(x).reshape(-1, N)[rows]
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= TOL
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        eng.input_projection(W, u, x)
    e0.record()
    for _ in range(20):
        eng.input_projection(W, u, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"input projection {T * B}x{N}x{Din}: {ms * 1e3:.1f} us, {2 * T * B * N * Din / ms / 1e9:.0f} TFLOP/s")


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["1", "2"])
def test_full_output_vs_torch_fp32(algo, monkeypatch):
    """Every element of the headline-sized projection against a torch fp32
    matmul of the same bf16 inputs, for both kernels (FRNN_WX_ALGO=1: 128x256
    single-CTA tiles; default: CTA-pair 256x256 persistent)."""
    import torch
    from paper_2412_07752_b200 import FlashRNN
    monkeypatch.setenv("FRNN_WX_ALGO", algo)
    T, B, Din, N = 1024, 16, 768, 3072
    g = torch.Generator(device="cuda").manual_seed(11)
    u = torch.randn(T, B, Din, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, Din, device="cuda", generator=g) / Din ** 0.5).bfloat16()
    x = FlashRNN().input_projection(W, u)
    ref = u.float().reshape(-1, Din) @ W.float().T
    got = x.float().reshape(-1, N)
    err = ((got - ref).norm() / ref.norm()).item()
    worst = ((got - ref).abs() / (ref.abs() + 1e-2)).max().item()
    assert err <= TOL, err
    assert worst <= 2 ** -7, worst   # each element within one bf16 rounding of the fp32 sum
