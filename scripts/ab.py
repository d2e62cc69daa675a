#!/usr/bin/env python3
"""Interleaved A/B timing of kernel variants selected by environment knobs
(read by the library at every launch), so that box-to-box and drift noise
cancels: each rep runs every setting once, medians reported per setting.

    python scripts/ab.py --set FRNN_PVEC=0 --set FRNN_PVEC=1 [--variant slstm --reps 15]
"""
import argparse
import os
import statistics as S
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2412_07752_b200 import FlashRNN  # noqa: E402

NS_NG = {"elman": (1, 1), "lstm": (2, 4), "gru": (1, 4), "slstm": (4, 4)}
ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="slstm")
ap.add_argument("--hidden", type=int, default=768)
ap.add_argument("--heads", type=int, default=1)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--seq", type=int, default=1024)
ap.add_argument("--reps", type=int, default=15)
ap.add_argument("--set", action="append", default=[], help="NAME=VAL[,NAME=VAL] one setting")
a = ap.parse_args()
sets = [dict(kv.split("=") for kv in s.split(",")) for s in (a.set or [""]) if s] or [{}]
NS, NG = NS_NG[a.variant]
DH = a.hidden // a.heads
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
R = (torch.randn(a.heads, NG, DH, DH, device=dev, generator=g) / DH ** 0.5).bfloat16()
b = (0.1 * torch.randn(NG, a.hidden, device=dev, generator=g)).bfloat16()
x = torch.randn(a.seq, a.batch, NG, a.hidden, device=dev, generator=g).bfloat16()
s0 = (0.5 * torch.randn(NS, a.batch, a.hidden, device=dev, generator=g)).bfloat16()
dsf = torch.randn(NS, a.batch, a.hidden, device=dev, generator=g).bfloat16()
eng = FlashRNN()
res = {i: ([], []) for i in range(len(sets))}
for rep in range(a.reps + 1):
    for i, st_env in enumerate(sets):
        for k, v in st_env.items():
            os.environ[k] = v
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        e0.record()
        st, ga = eng.forward(a.variant, R, b, x, s0)
        e1.record()
        eng.backward(a.variant, R, b, st, ga, dsf)
        e2.record()
        torch.cuda.synchronize()
        for k in st_env:
            del os.environ[k]
        if rep:
            res[i][0].append(1e3 * e0.elapsed_time(e1) / a.seq)
            res[i][1].append(1e3 * e1.elapsed_time(e2) / a.seq)
print(f"{a.variant} H={a.hidden} NH={a.heads} B={a.batch} T={a.seq}  us/step median (min)")
for i, st_env in enumerate(sets):
    f, bw = res[i]
    print(f"  {','.join(f'{k}={v}' for k, v in st_env.items()) or 'default':40s} fwd {S.median(f):.3f} ({min(f):.3f})"
          f"  bwd {S.median(bw):.3f} ({min(bw):.3f})")
