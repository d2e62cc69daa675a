#!/usr/bin/env python3
"""Run fwd+bwd of one configuration a few times (profiling driver for ncu).

    python scripts/run_case.py --variant slstm --hidden 3072 --batch 64 --seq 8 --reps 2
"""
import argparse
import os
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
ap.add_argument("--seq", type=int, default=16)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--algo", default="auto")
ap.add_argument("--time", action="store_true", help="print CUDA-event time per rep")
a = ap.parse_args()
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
for i in range(a.reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    import time
    torch.cuda.synchronize()
    e0.record()
    h0 = time.perf_counter()
    st, ga = eng.forward(a.variant, R, b, x, s0, algo=a.algo)
    h1 = time.perf_counter()
    e1.record()
    eng.backward(a.variant, R, b, st, ga, dsf, algo=a.algo)
    h2 = time.perf_counter()
    e2.record()
    torch.cuda.synchronize()
    if a.time:
        print(f"  host enqueue: fwd {1e3 * (h1 - h0):.3f} ms  bwd {1e3 * (h2 - h1):.3f} ms")
    if a.time:
        f, bw = e0.elapsed_time(e1), e1.elapsed_time(e2)
        print(f"rep {i}: fwd {f:.3f} ms ({1e3 * f / a.seq:.2f} us/step)  bwd {bw:.3f} ms ({1e3 * bw / a.seq:.2f} us/step)")
