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


def reduce_param_grads(dR, dbias, s: dict, dist, T=None, B=None, NH=None, DH=None) -> None:
    """In-place sum of dR / dbias over the ranks that share this rank's head
    range (the batch shards; engine.hpp:317, :327-330).  With mixed head x
    batch sharding every rank joins one torch.distributed subgroup per head
    partition (new_group is collective, so all ranks create all groups in the
    same order); pure batch sharding reduces over the whole world."""
    if not s["reduce_params"]:
        return
    world = dist.get_world_size()
    if NH is None:  # legacy call: only valid for pure batch sharding
        if s["head_begin"] != 0:
            raise ValueError("mixed head x batch sharding: pass T, B, NH, DH")
        dist.all_reduce(dR)
        dist.all_reduce(dbias)
        return
    shards = [shard_of(T, B, NH, DH, world, r) for r in range(world)]
    heads = sorted({(x["head_begin"], x["head_end"]) for x in shards})
    if len(heads) == 1:
        dist.all_reduce(dR)
        dist.all_reduce(dbias)
        return
    mine = None
    for hb in heads:  # every rank creates every group, in the same order
        g = dist.new_group([r for r, x in enumerate(shards) if (x["head_begin"], x["head_end"]) == hb])
        if hb == (s["head_begin"], s["head_end"]):
            mine = g
    dist.all_reduce(dR, group=mine)
    dist.all_reduce(dbias, group=mine)


class LibDist:
    """The library's own multi-GPU layer (include/flashrnn_dist.h): an NCCL
    communicator created by libflashrnn (dlopen'ed NCCL, no PyTorch on its
    data path), the fp32 dR/db reduction across batch shards and the
    activation gather.  `bootstrap` only ships the 128-byte NCCL unique id from
    rank 0 to the others (any torch.distributed process group will do)."""

    def __init__(self, world: int, rank: int, bootstrap=None):
        import ctypes as C

        import torch

        from .abi import load

        self.C, self.torch = C, torch
        self.world, self.rank = world, rank
        L = self.lib = load()
        vp = C.c_void_p
        L.frnn_dist_unique_id.argtypes = [C.c_char_p]
        L.frnn_dist_init.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.frnn_dist_destroy.argtypes = [vp]
        from .abi import Cell
        pc = C.POINTER(Cell)
        L.frnn_dist_workspace_size.argtypes = [vp, pc, _Shape(), C.c_int32, C.POINTER(C.c_size_t)]
        L.frnn_dist_reduce_param_grads.argtypes = [vp, pc, _Shape(), C.c_int32, vp, vp, vp, C.c_size_t, vp]
        L.frnn_dist_gather.argtypes = [vp, pc, _Shape(), C.c_int32, vp, vp, C.c_size_t, vp]
        idb = C.create_string_buffer(128)
        if rank == 0:
            _chk(L.frnn_dist_unique_id(idb))
        if world > 1:
            t = torch.tensor(list(idb.raw), dtype=torch.uint8)
            if bootstrap is not None and bootstrap.get_backend() == "nccl":
                t = t.cuda()
            bootstrap.broadcast(t, src=0)
            idb = C.create_string_buffer(bytes(t.cpu().tolist()), 128)
        self.handle = vp()
        _chk(L.frnn_dist_init(idb, world, rank, C.byref(self.handle)))
        self._ws = None

    def _workspace(self, cell, shape, dt, device):
        n = self.C.c_size_t()
        _chk(self.lib.frnn_dist_workspace_size(self.handle, self.C.byref(cell), shape, dt, self.C.byref(n)))
        if self._ws is None or self._ws.numel() < n.value:
            self._ws = self.torch.empty(max(256, n.value), dtype=self.torch.uint8, device=device)
        return self._ws

    def reduce_param_grads(self, variant, T, B, NH, DH, dR, dbias, stream=None):
        from .abi import DTYPE, Shape, cell_spec
        cell, shape = cell_spec(variant), Shape(T, B, NH, DH)
        dt = DTYPE["bf16"] if dR.dtype == self.torch.bfloat16 else DTYPE["f32"]
        ws = self._workspace(cell, shape, dt, dR.device)
        s = stream if stream is not None else self.torch.cuda.current_stream(dR.device).cuda_stream
        _chk(self.lib.frnn_dist_reduce_param_grads(self.handle, self.C.byref(cell), shape, dt, dR.data_ptr(),
                                                   dbias.data_ptr(), ws.data_ptr(), ws.numel(), s))

    def gather(self, variant, T, B, NH, DH, local: dict, full: dict, stream=None):
        """local/full: dicts with any of states, gates, dx, ds0, dR, dbias."""
        from .abi import DTYPE, Shape, cell_spec
        C = self.C
        names = ("states", "gates", "dx", "ds0", "dR", "dbias")
        ptr = [local[k].data_ptr() if k in local and k in full else None for k in names]
        fptr = [full[k].data_ptr() if k in local and k in full else None for k in names]
        tens = (C.c_void_p * 12)(*(ptr + fptr))
        cell, shape = cell_spec(variant), Shape(T, B, NH, DH)
        t0 = next(v for v in local.values())
        dt = DTYPE["bf16"] if t0.dtype == self.torch.bfloat16 else DTYPE["f32"]
        ws = self._workspace(cell, shape, dt, t0.device)
        s = stream if stream is not None else self.torch.cuda.current_stream(t0.device).cuda_stream
        _chk(self.lib.frnn_dist_gather(self.handle, C.byref(cell), shape, dt, C.cast(tens, C.c_void_p),
                                       ws.data_ptr(), ws.numel(), s))

    def close(self):
        if self.handle:
            self.lib.frnn_dist_destroy(self.handle)
            self.handle = self.C.c_void_p()


def _Shape():
    from .abi import Shape
    return Shape


def _chk(rc):
    from .abi import _check
    _check(rc)


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
