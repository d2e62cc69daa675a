"""Per-step stamps of the multi-cluster forward (frnn_debug_profile): local / remote h arrival, MMA halves, publish.

    python scripts/mc_profile.py 1024
"""
import ctypes as C, os, statistics as S, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2412_07752_b200 import FlashRNN
from paper_2412_07752_b200.abi import load
H = int(sys.argv[1]); T = 256
dev = torch.device("cuda", 0); g = torch.Generator(device=dev).manual_seed(0)
R = (torch.randn(1, 4, H, H, device=dev, generator=g) / H ** 0.5).bfloat16()
b = (0.1 * torch.randn(4, H, device=dev, generator=g)).bfloat16()
x = torch.randn(T, 16, 4, H, device=dev, generator=g).bfloat16()
s0 = (0.5 * torch.randn(2, 16, H, device=dev, generator=g)).bfloat16()
eng = FlashRNN(); L = load(); L.frnn_debug_profile.argtypes = [C.c_void_p, C.c_int32]
pf = eng.plan("lstm", T, 16, 1, H, "bf16", "forward"); grid = pf["grid"]
st, ga = eng.forward("lstm", R, b, x, s0)
buf = torch.zeros(grid * T * 8, dtype=torch.int64, device=dev)
L.frnn_debug_profile(buf.data_ptr(), T); eng.forward("lstm", R, b, x, s0, st, ga); torch.cuda.synchronize(); L.frnn_debug_profile(None, 0)
v = buf.view(grid, T, 8).cpu().tolist()
def med(f):
    q = sorted(f(c, t) for c in range(grid) for t in range(T // 4, 3 * T // 4)); return q[len(q)//2], q[len(q)//10], q[9*len(q)//10]
print("H", H, pf)
print("step", med(lambda c, t: v[c][t + 1][0] - v[c][t][0]))
print("local wait (0->1)", med(lambda c, t: v[c][t][1] - v[c][t][0]))
print("local MMAs + remote wait (1->5)", med(lambda c, t: v[c][t][5] - v[c][t][1]))
print("remote MMAs + done (5->2)", med(lambda c, t: v[c][t][2] - v[c][t][5]))
print("drain+pointwise (2->3)", med(lambda c, t: v[c][t][3] - v[c][t][2]))
print("publish (3->4)", med(lambda c, t: v[c][t][4] - v[c][t][3]))
print("publish(t) -> remote flag seen (4@t -> 6@t+1)", med(lambda c, t: v[c][t + 1][6] - v[c][t][4]))
print("remote flag seen -> remote data landed (6 -> 5 of t+1)", med(lambda c, t: v[c][t + 1][5] - v[c][t + 1][6]))
