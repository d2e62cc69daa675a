"""The library's multi-GPU layer (include/flashrnn_dist.h, csrc/dist.cu).

GPU (one B200 here): the NCCL communicator at world 1, the fp32 round trip
of the dR/db reduction (FRNN_DIST_FORCE_REDUCE runs the collective even
without batch shards: bf16 -> fp32 -> allreduce -> bf16 must be exact), the
gather at world 1, and the placement half of the gather for 2..8-rank
layouts (pure batch, pure head, mixed head x batch, ragged batch) emulated on
one device: each rank's shard is cut from a full tensor by frnn_partition,
packed as ncclAllGather would deliver it, placed back, and must reproduce the
full tensor bit for bit.  The multi-rank NCCL calls themselves run in
bench.py under torchrun (no multi-GPU box in this environment).
"""
import ctypes as C
import os

import pytest

pytestmark = pytest.mark.gpu

NAMES = ("states", "gates", "dx", "ds0", "dR", "dbias")


def _shapes(v, T, B, NH, DH):
    from paper_2412_07752_b200.abi import cell_spec
    c = cell_spec(v)
    NS, NG, D = c.num_states, c.num_gates, NH * DH
    return {"states": (T + 1, NS, B, D), "gates": (T, NG, B, D), "dx": (T, B, NG, D), "ds0": (NS, B, D),
            "dR": (NH, NG, DH, DH), "dbias": (NG, D)}


def _local(name, full, s, DH):
    bs, es = slice(s["batch_begin"], s["batch_end"]), slice(s["head_begin"] * DH, s["head_end"] * DH)
    hs = slice(s["head_begin"], s["head_end"])
    return {"states": lambda t: t[:, :, bs, es], "gates": lambda t: t[:, :, bs, es],
            "dx": lambda t: t[:, bs, :, es], "ds0": lambda t: t[:, bs, es],
            "dR": lambda t: t[hs], "dbias": lambda t: t[:, es]}[name](full).contiguous()


@pytest.mark.parametrize("v,T,B,NH,DH,world", [
    ("lstm", 5, 16, 1, 64, 2),     # pure batch sharding (the weak-scaling layout)
    ("slstm", 4, 16, 1, 32, 8),
    ("gru", 3, 5, 1, 32, 2),       # ragged batch split (3 + 2 rows)
    ("lstm", 3, 4, 4, 16, 4),      # pure head sharding
    ("lstm", 3, 6, 4, 16, 8),      # mixed: 4 head partitions x 2 batch partitions
    ("elman", 2, 7, 12, 8, 6),     # mixed, ragged
])
def test_gather_placement(v, T, B, NH, DH, world):
    import torch
    from paper_2412_07752_b200.abi import DTYPE, Shape, cell_spec, load, partition
    L = load()
    L.frnn_debug_dist_place.argtypes = [C.c_void_p, Shape, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_size_t), C.c_void_p]
    cell = cell_spec(v)
    shards = [partition(T, B, NH, DH, world, r) for r in range(world)]
    for k, name in enumerate(NAMES):
        shp = _shapes(v, T, B, NH, DH)[name]
        full = torch.randint(-30000, 30000, shp, dtype=torch.int16, device="cuda").view(torch.bfloat16)
        blk = C.c_size_t()
        assert L.frnn_debug_dist_place(C.byref(cell), Shape(T, B, NH, DH), DTYPE["bf16"], world, k, None, None,
                                       C.byref(blk), None) == 0
        stage = torch.zeros(world, blk.value, dtype=torch.bfloat16, device="cuda")
        for r, s in enumerate(shards):
            loc = _local(name, full, s, DH).reshape(-1)
            stage[r, :loc.numel()] = loc
        out = torch.zeros_like(full)
        assert L.frnn_debug_dist_place(C.byref(cell), Shape(T, B, NH, DH), DTYPE["bf16"], world, k,
                                       stage.data_ptr(), out.data_ptr(), C.byref(blk), None) == 0
        torch.cuda.synchronize()
        if name in ("dR", "dbias"):  # every head partition placed once (from its batch shard 0)
            assert torch.equal(out.view(torch.int16), full.view(torch.int16)), name
        else:
            assert torch.equal(out.view(torch.int16), full.view(torch.int16)), name


def test_nccl_world1_reduce_and_gather(monkeypatch):
    import torch
    from paper_2412_07752_b200 import FlashRNN
    from paper_2412_07752_b200.distributed import LibDist
    d = LibDist(1, 0)
    assert d.lib.frnn_dist_nccl_version() > 0
    eng = FlashRNN()
    T, B, NH, DH, v = 6, 16, 2, 64, "lstm"
    g = torch.Generator(device="cuda").manual_seed(0)
    R = (torch.randn(NH, 4, DH, DH, device="cuda", generator=g) / 8).bfloat16()
    b = (0.1 * torch.randn(4, NH * DH, device="cuda", generator=g)).bfloat16()
    x = torch.randn(T, B, 4, NH * DH, device="cuda", generator=g).bfloat16()
    s0 = (0.5 * torch.randn(2, B, NH * DH, device="cuda", generator=g)).bfloat16()
    dsf = torch.randn(2, B, NH * DH, device="cuda", generator=g).bfloat16()
    st, ga = eng.forward(v, R, b, x, s0)
    out = eng.backward(v, R, b, st, ga, dsf)
    dR0, db0 = out["dR"].clone(), out["dbias"].clone()
    monkeypatch.setenv("FRNN_DIST_FORCE_REDUCE", "1")
    d.reduce_param_grads(v, T, B, NH, DH, out["dR"], out["dbias"])
    torch.cuda.synchronize()
    assert torch.equal(out["dR"], dR0) and torch.equal(out["dbias"], db0)  # fp32 round trip is exact
    local = {"states": st, "gates": ga, "dx": out["dx"], "ds0": out["ds0"], "dR": out["dR"], "dbias": out["dbias"]}
    full = {k: torch.zeros_like(t) for k, t in local.items()}
    d.gather(v, T, B, NH, DH, local, full)
    torch.cuda.synchronize()
    for k in local:
        assert torch.equal(full[k], local[k]), k
    d.close()
