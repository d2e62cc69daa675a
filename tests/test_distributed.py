"""Multi-process (gloo, world_size 2, CPU) test of the batch x head sharded path.

Each rank slices the full inputs to its frnn_partition shard, runs the
per-shard recurrence (the CPU oracle stands in for the GPU kernels here -- the
host-side slicing / gather / reduction logic is what is under test), and
reassembles full outputs with paper_2412_07752_b200.distributed; the result
must equal the unsharded oracle run exactly (float64, same summation per
shard up to the cross-shard dR/db sum).
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, variant, T, B, NH, DH, q):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import torch
        import torch.distributed as dist

        import oracle as O
        from paper_2412_07752_b200 import distributed as PD

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        orc = O.Oracle()
        full = {k: torch.from_numpy(v) for k, v in orc.generate(variant, T, B, NH, DH, seed=9).items()}
        full["d_hidden"] = torch.from_numpy(np.random.RandomState(3).randn(T, B, NH * DH))
        s = PD.shard_of(T, B, NH, DH, world, rank)
        loc = PD.local_inputs(full, s, DH)
        st, ga = orc.forward(variant, loc["R"].numpy(), loc["bias"].numpy(), loc["x"].numpy(), loc["s0"].numpy())
        g = orc.backward(variant, loc["R"].numpy(), st, ga, loc["dsf"].numpy(), "value", 0.5,
                         loc["d_hidden"].numpy())
        local = {"states": torch.from_numpy(st), "gates": torch.from_numpy(ga)}
        local.update({k: torch.from_numpy(v) for k, v in g.items()})
        out = PD.gather_outputs(local, s, world, T, B, NH, DH, dist)
        if rank == 0:
            st0, ga0 = orc.forward(variant, *(full[k].numpy() for k in ("R", "bias", "x", "s0")))
            g0 = orc.backward(variant, full["R"].numpy(), st0, ga0, full["dsf"].numpy(), "value", 0.5,
                              full["d_hidden"].numpy())
            ref = {"states": st0, "gates": ga0, **g0}
            errs = {k: float(np.max(np.abs(out[k].numpy() - ref[k]))) for k in ref}
            q.put(errs)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures to the test
        q.put({"error": repr(e)})


@pytest.mark.parametrize("variant,B,NH", [("lstm", 6, 1), ("slstm", 5, 2), ("gru", 4, 4)])
def test_sharded_matches_unsharded(variant, B, NH):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    T, DH, world = 5, 8, 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, variant, T, B, NH, DH, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert "error" not in res, res
    for k, e in res.items():
        # activations are bit-identical; dR/db differ only by the cross-shard sum order
        assert e <= (1e-12 if k in ("dR", "dbias") else 0.0), (k, e)
