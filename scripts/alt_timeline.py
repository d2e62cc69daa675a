#!/usr/bin/env python3
"""Per-step timeline of the alternating-path kernels from globaltimer stamps
(frnn_debug_profile): [launch][cta][start, dependency released, GEMM done, end].

    python scripts/alt_timeline.py --hidden 3072 --batch 64 --seq 64 --steps 32
"""
import argparse
import ctypes as C
import os
import statistics as S
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_07752_b200 import FlashRNN  # noqa: E402
from paper_2412_07752_b200.abi import load  # noqa: E402

NS_NG = {"elman": (1, 1), "lstm": (2, 4), "gru": (1, 4), "slstm": (4, 4)}
ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="slstm")
ap.add_argument("--hidden", type=int, default=3072)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--seq", type=int, default=64)
ap.add_argument("--steps", type=int, default=32)
a = ap.parse_args()
NS, NG = NS_NG[a.variant]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
DH = a.hidden
R = (torch.randn(1, NG, DH, DH, device=dev, generator=g) / DH ** 0.5).bfloat16()
b = (0.1 * torch.randn(NG, DH, device=dev, generator=g)).bfloat16()
x = torch.randn(a.seq, a.batch, NG, DH, device=dev, generator=g).bfloat16()
s0 = (0.5 * torch.randn(NS, a.batch, DH, device=dev, generator=g)).bfloat16()
dsf = torch.randn(NS, a.batch, DH, device=dev, generator=g).bfloat16()
eng = FlashRNN()
L = load()
L.frnn_debug_profile.argtypes = [C.c_void_p, C.c_int32]


def timeline(name, grid, run):
    buf = torch.zeros(a.steps * grid * 8, dtype=torch.int64, device=dev)
    L.frnn_debug_profile(buf.data_ptr(), a.steps)
    run()
    torch.cuda.synchronize()
    L.frnn_debug_profile(None, 0)
    v = buf.view(a.steps, grid, 8).cpu().tolist()
    rows = []
    for k in range(a.steps):
        st = [c[0] for c in v[k]]
        rel = [c[1] for c in v[k]]
        dn = [c[2] for c in v[k]]
        en = [c[3] for c in v[k]]
        pr = [c[4] for c in v[k]]
        p5 = [c[5] for c in v[k]]
        p6 = [c[6] for c in v[k]]
        p7 = [c[7] for c in v[k]]
        rows.append(dict(s0=min(st), s1=max(st), r0=min(rel), r1=max(rel), d=S.median([d - r for d, r in zip(dn, rel)]),
                         prod=S.median([q - r for q, r in zip(pr, rel)]) if min(pr) > 0 else -1,
                         p5=S.median([q - r for q, r in zip(p5, rel)]) if min(p5) > 0 else -1,
                         p6=S.median([q - r for q, r in zip(p6, p5)]) if min(p6) > 0 else -1,
                         p7=S.median([q - r for q, r in zip(p7, p5)]) if min(p7) > 0 else -1,
                         dmax=max(d - r for d, r in zip(dn, rel)), ep=S.median([e - d for e, d in zip(en, dn)]),
                         e1=max(en), e0=min(en)))
    print(f"== {name}: grid {grid}, ns")
    print(" step  start-prevEnd  release-prevEnd  release spread  producer(med)  gemm(med/max)  epilogue(med)  kernel(start..end)")
    for k in range(1, a.steps):
        p, c = rows[k - 1], rows[k]
        print(f" {k:4d}  {c['s0'] - p['e1']:8d}  {c['r0'] - p['e1']:8d}  {c['r1'] - c['r0']:8d}  {c['prod']:8.0f}  {c['d']:7.0f}/{c['dmax']:7.0f}  {c['ep']:7.0f}  {c['e1'] - c['s0']:8d}"
              f"  step period {c['e1'] - p['e1']}  producer release->own wait {c['p5']:.0f}  first empty wait {c['p6']:.0f}  mma warp stage-0 done after release {c['p7']:.0f}")


pf = eng.plan(a.variant, a.seq, a.batch, 1, DH, "bf16", "forward")
pb = eng.plan(a.variant, a.seq, a.batch, 1, DH, "bf16", "backward")
st, ga = eng.forward(a.variant, R, b, x, s0)
eng.backward(a.variant, R, b, st, ga, dsf)
torch.cuda.synchronize()
timeline("forward", pf["grid"], lambda: eng.forward(a.variant, R, b, x, s0, st, ga))
timeline("backward", pb["grid"], lambda: eng.backward(a.variant, R, b, st, ga, dsf))
