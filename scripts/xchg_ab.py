#!/usr/bin/env python3
"""A/B of the backward partial-exchange variants (FRNN_XCHG=0/1/2) on the
cluster kernels: per-step backward time, normal and synchronisation skeleton.

    for x in 0 1 2; do FRNN_XCHG=$x python scripts/xchg_ab.py; done
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_07752_b200 import FlashRNN  # noqa: E402
from paper_2412_07752_b200.abi import load  # noqa: E402

variant = sys.argv[1] if len(sys.argv) > 1 else "slstm"
NS, NG = {"slstm": (4, 4), "lstm": (2, 4), "gru": (1, 4), "elman": (1, 1)}[variant]
T, B, DH = 1024, 16, 768
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
R = (torch.randn(1, NG, DH, DH, device=dev, generator=g) / DH ** 0.5).bfloat16()
b = (0.1 * torch.randn(NG, DH, device=dev, generator=g)).bfloat16()
x = torch.randn(T, B, NG, DH, device=dev, generator=g).bfloat16()
s0 = (0.5 * torch.randn(NS, B, DH, device=dev, generator=g)).bfloat16()
dsf = torch.randn(NS, B, DH, device=dev, generator=g).bfloat16()
eng = FlashRNN()
L = load()
L.frnn_debug_skeleton.argtypes = [C.c_int32]
st, ga = eng.forward(variant, R, b, x, s0)
ref = eng.backward(variant, R, b, st, ga, dsf)
ref = {k: v.clone() for k, v in ref.items()}
out = {}
for skel in (0, 1):
    L.frnn_debug_skeleton(skel)
    best = 1e9
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr = eng.backward(variant, R, b, st, ga, dsf)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[skel] = 1e3 * best / T
    if skel == 0:
        same = all(torch.equal(gr[k], ref[k]) for k in gr)
L.frnn_debug_skeleton(0)
print(f"FRNN_XCHG={os.environ.get('FRNN_XCHG', 'default')} {variant}: bwd {out[0]:.2f} us/step, "
      f"skeleton {out[1]:.2f} us/step, deterministic={same}")
