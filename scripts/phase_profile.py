#!/usr/bin/env python3
"""Per-step phase breakdown (clock64 stamps, frnn_debug_profile) of the
cluster-resident fused kernels.

    python scripts/phase_profile.py [--variant slstm --heads 1 --hidden 768 --batch 16 --seq 256]

Forward stamps: 0 step start, 1 h(t) arrived + MMA issued, 2 MMA done,
3 pointwise done, 4 h(t+1) published.  Backward: 0 start, 1 partials of
step t+1 absorbed, 2 Jacobian done (MMA issue), 3 MMA done, 4 partials out.
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
ap.add_argument("--heads", type=int, default=1)
ap.add_argument("--hidden", type=int, default=768)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--seq", type=int, default=256)
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
L = load()
if os.environ.get("FRNN_DEBUG_SKELETON"):  # synchronisation skeleton only (results are garbage)
    L.frnn_debug_skeleton.argtypes = [C.c_int32]
    L.frnn_debug_skeleton(1)
L.frnn_debug_profile.argtypes = [C.c_void_p, C.c_int32]
pf = eng.plan(a.variant, a.seq, a.batch, a.heads, DH, "bf16", "forward")
pb = eng.plan(a.variant, a.seq, a.batch, a.heads, DH, "bf16", "backward")
print(a.variant, a.heads, DH, {k: pf[k] for k in ("algo", "cluster", "rows_per_cta", "grid", "threads")})
st, ga = eng.forward(a.variant, R, b, x, s0)
eng.backward(a.variant, R, b, st, ga, dsf)
torch.cuda.synchronize()


def profile(name, grid, run, labels, extra=(), cross=()):
    buf = torch.zeros(grid * a.seq * 8, dtype=torch.int64, device=dev)
    L.frnn_debug_profile(buf.data_ptr(), a.seq)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    L.frnn_debug_profile(None, 0)
    v = buf.view(grid, a.seq, 8).cpu().tolist()
    ms = e0.elapsed_time(e1)
    lo, hi = a.seq // 4, 3 * a.seq // 4
    per = []
    for k in range(len(labels)):
        vals = []
        for c in range(grid):
            for t in range(lo, hi):
                nxt = v[c][t + 1][0] if k == len(labels) - 1 else v[c][t][k + 1]
                vals.append(nxt - v[c][t][k])
        per.append(vals)
    step = [v[c][t + 1][0] - v[c][t][0] for c in range(grid) for t in range(lo, hi)]
    print(f"  {name}: {ms:.2f} ms total, {1e3 * ms / a.seq:.2f} us/step; ctas={grid}; step cycles {S.median(step):.0f}")
    for lab, vals in zip(labels, per):
        q = sorted(vals)
        print(f"   {lab:>26s}: {S.median(vals):8.0f} {q[len(q) // 10]:8.0f} {q[9 * len(q) // 10]:8.0f}   (median p10 p90)")
    for lab, k0, k1 in extra:  # stamp k1 - stamp k0 of the same step (thread 0)
        q = sorted(v[c][t][k1] - v[c][t][k0] for c in range(grid) for t in range(lo, hi))
        print(f"   {lab:>26s}: {q[len(q) // 2]:8.0f} {q[len(q) // 10]:8.0f} {q[9 * len(q) // 10]:8.0f}   (median p10 p90)")
    for lab, k0, k1 in cross:  # stamp k1 of step t+1 - stamp k0 of step t (same CTA)
        q = sorted(v[c][t + 1][k1] - v[c][t][k0] for c in range(grid) for t in range(lo, hi))
        print(f"   {lab:>26s}: {q[len(q) // 2]:8.0f} {q[len(q) // 10]:8.0f} {q[9 * len(q) // 10]:8.0f}   (median p10 p90)")


profile("fwd", pf["grid"], lambda: eng.forward(a.variant, R, b, x, s0, st, ga),
        ["wait h + MMA issue", "trace(t-1)+x prefetch+MMA", "tmem->xs+pointwise", "publish(multicast)",
         "loop"],
        [("  of which tmem->xs+sync", 2, 5), ("  of which cell math", 5, 6), ("  of which h slice+sync", 6, 3)])
profile("bwd", pb["grid"], lambda: eng.backward(a.variant, R, b, st, ga, dsf),
        ["absorb(wait+load+sum)", "jacobian", "mma", "partials out+arrive", "dx stores"],
        [("  issue -> last block done", 2, 6), ("  last block drained+pushed", 6, 7),
         ("  of absorb: sum+clip", 5, 1)],
        # critical path across CTAs: last warp's pushes of step k (slot 7) -> the
        # partials of step k complete at thread 0 of every CTA (slot 5 of step k+1)
        [("  pushes -> arrival (same CTA)", 7, 5)])
