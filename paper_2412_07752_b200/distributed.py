"""Batch x head sharding of the recurrence across GPUs.

Heads never mix (engine.hpp:139-142) and batch rows are independent except for
the sums over b in dR and db (engine.hpp:317, :327-330), so each rank runs the
full T loop on its own (batch, head) shard with NO per-step communication.
After the run:
  * states / gates / dx / ds0 are all-gathered along the sharded axes;
  * dR and db are sum-reduced across batch shards (all_reduce) and gathered
    across head shards (disjoint slices).
The shard map comes from the C ABI (frnn_partition).  Tensors are torch
tensors in rnnkit layouts; the collectives are torch.distributed (NCCL on
GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from .abi import partition


def shard_of(T, B, NH, DH, world, rank):
    return partition(T, B, NH, DH, world, rank)


def _eslice(s, DH):
    return slice(s["head_begin"] * DH, s["head_end"] * DH)


def local_inputs(full: dict, s: dict, DH: int) -> dict:
    """Slice full inputs (R, bias, x, s0, dsf[, d_hidden]) to one shard."""
    bs = slice(s["batch_begin"], s["batch_end"])
    es = _eslice(s, DH)
    hs = slice(s["head_begin"], s["head_end"])
    out = {
        "R": full["R"][hs].contiguous(),
        "bias": full["bias"][:, es].contiguous(),
        "x": full["x"][:, bs, :, es].contiguous(),
        "s0": full["s0"][:, bs, es].contiguous(),
        "dsf": full["dsf"][:, bs, es].contiguous(),
    }
    if full.get("d_hidden") is not None:
        out["d_hidden"] = full["d_hidden"][:, bs, es].contiguous()
    return out


def gather_outputs(local: dict, s: dict, world: int, T: int, B: int, NH: int, DH: int, dist) -> dict:
    """Reassemble full-size outputs on every rank from per-shard outputs.

    local: states [T+1][NS][b][e], gates [T][NG][b][e], dx [T][b][NG][e],
           ds0 [NS][b][e], dR [h][NG][DH][DH], dbias [NG][e]  (b, e, h local).
    """
    import torch

    shards = [shard_of(T, B, NH, DH, world, r) for r in range(world)]
    out = {}
    # batch/head-sharded activations: gather every rank's block, place by shard
    layouts = {"states": (2, 3), "gates": (2, 3), "dx": (1, 3), "ds0": (1, 2)}
    for name, (bdim, edim) in layouts.items():
        if name not in local:
            continue
        t = local[name]
        full_shape = list(t.shape)
        full_shape[bdim], full_shape[edim] = B, NH * DH
        blocks = _all_gather_var(t, dist, world)
        full = torch.zeros(full_shape, dtype=t.dtype, device=t.device)
        for r, blk in enumerate(blocks):
            sr = shards[r]
            idx = [slice(None)] * t.dim()
            idx[bdim] = slice(sr["batch_begin"], sr["batch_end"])
            idx[edim] = _eslice(sr, DH)
            full[tuple(idx)] = blk
        out[name] = full
    # parameter gradients: sum across batch shards, place head slices
    for name in ("dR", "dbias"):
        if name not in local:
            continue
        t = local[name]
        blocks = _all_gather_var(t, dist, world)
        if name == "dR":
            full = torch.zeros((NH,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        else:
            full = torch.zeros((t.shape[0], NH * DH), dtype=t.dtype, device=t.device)
        for r, blk in enumerate(blocks):
            sr = shards[r]
            if name == "dR":
                full[sr["head_begin"]:sr["head_end"]] += blk
            else:
                full[:, _eslice(sr, DH)] += blk
        out[name] = full
    return out


def reduce_param_grads(dR, dbias, s: dict, dist) -> None:
    """In-place data-parallel reduction used when every rank holds all heads
    (pure batch sharding, the benchmark's weak-scaling layout)."""
    if s["reduce_params"] and s["head_begin"] == 0:
        dist.all_reduce(dR)
        dist.all_reduce(dbias)


def _all_gather_var(t, dist, world):
    """all_gather for per-rank tensors whose shapes may differ (ragged shards)."""
    import torch

    shape = torch.tensor(list(t.shape), dtype=torch.int64, device=t.device)
    shapes = [torch.zeros_like(shape) for _ in range(world)]
    dist.all_gather(shapes, shape)
    flat = t.reshape(-1)
    n = max(int(torch.prod(s_)) for s_ in shapes)
    buf = torch.zeros(n, dtype=t.dtype, device=t.device)
    buf[: flat.numel()] = flat
    bufs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf)
    return [b[: int(torch.prod(s_))].reshape([int(x) for x in s_]) for b, s_ in zip(bufs, shapes)]
