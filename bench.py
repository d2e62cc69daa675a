#!/usr/bin/env python3
"""bench.py -- FlashRNN-B200 headline benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one forward + backward pass of the recurrence (rnnkit forward +
backward, engine.hpp:144/:222) over one batch: sLSTM, bf16, B=16 per GPU,
T=1024, H=768, NH=1 (BASELINE configs[1], the metric's workload), synthetic
inputs drawn on the device with the reference generator's distributions
(random_init.hpp:10-40).  Multi-GPU (torchrun, one rank per GPU, NCCL): weak
scaling -- every rank runs its own B=16 shard (frnn_partition batch sharding)
with no per-step communication, then dR/db are sum-reduced (the only
collective) inside the timed step.

value    device time (CUDA events on the launching stream) of K steps with
         inputs resident in HBM; L2 flushed (256 MB write) between timed steps;
         max over ranks; B*T*N / s.
e2e      the same metric through the C ABI with HOST buffers: pinned inputs
         (R, b, x, s0, dL/ds_T) copied H2D and the parameter gradients + ds0
         copied D2H inside the timed region, every step (the H2D of step i+1
         overlaps step i on a copy stream, double-buffered).
roofline the dominant kernel (largest share of the step), timed live with CUDA
         events on its launch stream (frnn_debug_kernel_ms); algorithmic FLOPs
         per launch = 2*NG_rec*NH*DH^2*B*T (its contraction); peak = measured
         sustained bf16 (MEASURED_PEAKS.json).
cpu_baseline  the unmodified reference engine (oracle/_ref, engine<float>)
         on this host, batch rows sharded over processes, bounded T sample.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sLSTM/LSTM fwd+bwd batch·timesteps/sec at B16 T1024 H768, 1/2/4/8 B200"
UNIT = "batch*timesteps/s"
NS_NG = {"elman": (1, 1), "lstm": (2, 4), "gru": (1, 4), "slstm": (4, 4)}
NGREC = {"elman": 1, "lstm": 4, "gru": 3, "slstm": 4}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--variant", default="slstm", choices=list(NS_NG))
    ap.add_argument("--heads", type=int, default=1)
    ap.add_argument("--hidden", type=int, default=768)
    ap.add_argument("--batch", type=int, default=16,
                    help="batch rows per GPU (weak scaling) or in total (strong scaling)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: B rows per GPU (global B = B x N); strong: global B fixed, sharded over the N GPUs")
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-steps", type=int, default=64)
    return ap.parse_args()


def workload_name(a, algo=None):
    path = {1: " (fused kernel, R resident on-chip)", 2: " (alternating path, R streamed from L2 every step)"}
    bdesc = f"B={a.batch} total" if getattr(a, "scaling", "weak") == "strong" else f"B={a.batch}/GPU"
    return (f"{a.variant} fwd+bwd bf16, {bdesc}, T={a.seq}, H={a.hidden}, NH={a.heads}"
            + path.get(algo, ""))


def flops_per_pass(a):
    """Algorithmic FLOPs of one recurrence contraction pass (fwd R.h, bwd R^T.dg,
    or dR): 2 * NG_rec * NH * DH^2 per batch-timestep (planner.cpp:404-416)."""
    dh = a.hidden // a.heads
    return 2.0 * NGREC[a.variant] * a.heads * dh * dh * a.batch * a.seq


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    (pynvml) polled every 5 ms on a background thread; nvidia-smi -lms 100 as
    the fallback when NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.thread = None

    def start(self):
        try:
            import threading

            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            self.sm, self.reasons, self.stop_flag = [], set(), threading.Event()

            def poll():
                while not self.stop_flag.is_set():
                    self.sm.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.reasons.update(k for k, b in bits.items() if r & b)
                    time.sleep(0.005)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join()
            return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.smax,
                    "reasons": sorted(self.reasons), "samples": len(self.sm), "source": "nvml, 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                               f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


def make_inputs(torch, dev, a, seed):
    """Synthetic inputs with the reference generator's distributions
    (random_init.hpp:10-40): R ~ N(0, 1/DH), b ~ N(0, 0.1^2), x ~ N(0,1),
    s0 ~ N(0, 0.5^2) (sLSTM n0 = 1 + 0.1|.|, m0 = 0), dL/ds_T ~ N(0,1)."""
    ns, ng = NS_NG[a.variant]
    nh, dh, B, T = a.heads, a.hidden // a.heads, a.batch, a.seq
    D = nh * dh
    g = torch.Generator(device=dev).manual_seed(seed)
    R = (torch.randn(nh, ng, dh, dh, device=dev, generator=g) / dh ** 0.5).bfloat16()
    b = (0.1 * torch.randn(ng, D, device=dev, generator=g)).bfloat16()
    x = torch.randn(T, B, ng, D, device=dev, generator=g).bfloat16()
    s0 = 0.5 * torch.randn(ns, B, D, device=dev, generator=g)
    if a.variant == "slstm":
        s0[2] = 1 + 0.1 * s0[2].abs()
        s0[3] = 0
    s0 = s0.bfloat16()
    dsf = torch.randn(ns, B, D, device=dev, generator=g).bfloat16()
    return dict(R=R, bias=b, x=x, s0=s0, dsf=dsf)


# ----------------------------------------------------------- CPU baseline ----
def _ref_worker(args):
    """One batch row through the unmodified reference engine<float>."""
    variant, T, DH, NH, seed = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O
    ref = O.Reference()
    ns, ng = NS_NG[variant]
    rng = np.random.RandomState(seed)
    D = NH * DH
    R = (rng.randn(NH, ng, DH, DH) / DH ** 0.5).astype(np.float32)
    b = (0.1 * rng.randn(ng, D)).astype(np.float32)
    x = rng.randn(T, 1, ng, D).astype(np.float32)
    s0 = (0.5 * rng.randn(ns, 1, D)).astype(np.float32)
    if variant == "slstm":
        s0[2] = 1 + 0.1 * np.abs(s0[2])
        s0[3] = 0
    dsf = rng.randn(ns, 1, D).astype(np.float32)
    t0 = time.perf_counter()
    st, ga = ref.forward(variant, R, b, x, s0, dtype=np.float32)
    ref.backward(variant, R, b, x, s0, st, ga, dsf, dtype=np.float32)
    return time.perf_counter() - t0


def cpu_reference_step(a, T_sample, pool, cores, B=None):
    """One bounded sample of the workload on the host: the B rows are
    independent (engine.hpp:173, only dR/db sum over b), so each row is one
    reference call in its own process; returns (B*T/s, wall seconds)."""
    B = a.batch if B is None else B
    jobs = [(a.variant, T_sample, a.hidden // a.heads, a.heads, 1000 + r) for r in range(B)]
    t0 = time.perf_counter()
    list(pool.map(_ref_worker, jobs))
    wall = time.perf_counter() - t0
    return B * T_sample / wall, wall


def make_pool(a, B=None):
    import concurrent.futures as cf
    import multiprocessing as mp
    cores = max(1, min(os.cpu_count() or 1, a.batch if B is None else B))
    return cf.ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("fork")), cores


def cpu_baseline(a):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.Reference.available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref/libref.so not built"}
    pool, cores = make_pool(a)
    try:
        cpu_reference_step(a, 2, pool, cores)  # warm the workers
        v, wall = cpu_reference_step(a, a.cpu_sample_steps, pool, cores)
    finally:
        pool.shutdown()
    return {"value": v, "unit": UNIT, "cores": cores, "host_cores": os.cpu_count(), "kind": "reference",
            "sample": (f"unmodified rnnkit engine<float> fwd+bwd, {a.variant} H={a.hidden} NH={a.heads}, "
                       f"B={a.batch} rows (one process each), T={a.cpu_sample_steps} steps, wall {wall:.2f} s"),
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(a, rank, world):
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref.so missing"}), flush=True)
        return
    # the same workload as our arm: B = batch_per_gpu x world rows (weak scaling),
    # each step a bounded T sample (shortened as rows grow, so the run stays minutes long)
    B = a.batch * world
    pool, cores = make_pool(a, B)
    T_s = max(8, a.cpu_sample_steps // world)
    try:
        for _ in range(a.warmup):
            cpu_reference_step(a, max(2, T_s // 8), pool, cores, B)
        walls = []
        for _ in range(a.steps):
            _, w = cpu_reference_step(a, T_s, pool, cores, B)
            walls.append(w)
    finally:
        pool.shutdown()
    total = sum(walls)
    value = B * T_s * a.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * total / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy RNG, reference distributions)",
        "config": {"workload": workload_name(a).replace(" bf16,", " (reference engine<float>, fp32 arithmetic),"),
                   "batch_per_gpu": a.batch, "global_batch": B, "seq_len": a.seq,
                   "hidden": a.hidden, "heads": a.heads, "sample_seq_len": T_s},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "host_cores": os.cpu_count(), "kind": "reference",
                         "sample": f"B={B} rows x T={T_s} steps per step, engine<float>",
                         "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- our impl ----
def e2e_shim(a):
    """The same fwd+bwd through the C++ drop-in with VALUE semantics, as an
    rnnkit caller uses it (tools/e2e_bench.cpp: host std::vector<BFloat16> in,
    host vectors out, every conversion and copy inside the host wall-clock
    timing).  Built on first use; None when the toolchain is missing."""
    exe = os.path.join(ROOT, "build", "e2e_bench")
    src = os.path.join(ROOT, "tools", "e2e_bench.cpp")
    try:
        if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
            from paper_2412_07752_b200.build import build_tool
            build_tool("e2e_bench")
        r = subprocess.run([exe, "--variant", a.variant, "--hidden", str(a.hidden), "--heads", str(a.heads),
                            "--batch", str(a.batch), "--seq", str(a.seq), "--steps", "4", "--warmup", "2"],
                           capture_output=True, text=True, timeout=600)
        if r.returncode != 0:
            return {"unavailable": (r.stderr or r.stdout).strip()[-300:]}
        d = json.loads(r.stdout.strip().splitlines()[-1])
        return {"value": d["value"], "unit": UNIT, "ms_per_step": d["ms_per_step"],
                "h2d_bytes_per_step": d["h2d_bytes_per_step"], "d2h_bytes_per_step": d["d2h_bytes_per_step"],
                "host_threads": d["host_threads"],
                "api": "flashrnn::rnn::forward/backward (include/flashrnn/engine.hpp), host vectors, "
                       "host wall clock (tools/e2e_bench.cpp)"}
    except Exception as e:  # the headline numbers stand without it
        return {"unavailable": f"{type(e).__name__}: {e}"[:300]}


def run_ours(a, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2412_07752_b200 import FlashRNN
    from paper_2412_07752_b200.abi import load, partition

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    eng = FlashRNN()
    L = load()
    L.frnn_debug_timing.argtypes = [C.c_int32]
    L.frnn_debug_launches.argtypes = [C.POINTER(C.c_int64)]
    L.frnn_debug_kernel_ms.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    # the rank's (batch x head) shard of the global problem (frnn_partition); every
    # kernel below runs on the LOCAL shape, the metric counts the global one
    DH = a.hidden // a.heads
    global_B = a.batch * world if a.scaling == "weak" else a.batch
    shard = partition(a.seq, global_B, a.heads, DH, world, rank)
    ga_ = argparse.Namespace(**vars(a))  # global view (names, FLOP accounting)
    a = argparse.Namespace(**vars(a))
    a.batch = shard["batch_end"] - shard["batch_begin"]
    a.heads = shard["head_end"] - shard["head_begin"]
    a.hidden = a.heads * DH
    libdist = None
    share = os.environ.get("FRNN_BENCH_SHARE_GPU") == "1"  # test hook: ranks share cuda:0 (gloo, no NCCL)
    if world > 1 and not share:  # the library's own NCCL layer (include/flashrnn_dist.h); torch ships the NCCL id
        from paper_2412_07752_b200.distributed import LibDist
        libdist = LibDist(world, rank, bootstrap=dist)
    inp = make_inputs(torch, dev, a, seed=rank)
    ns, ng = NS_NG[a.variant]
    D = a.hidden
    st = torch.empty(a.seq + 1, ns, a.batch, D, dtype=torch.bfloat16, device=dev)
    ga = torch.empty(a.seq, ng, a.batch, D, dtype=torch.bfloat16, device=dev)
    out = dict(dx=torch.empty_like(inp["x"]), dbias=torch.empty_like(inp["bias"]),
               dR=torch.empty_like(inp["R"]), ds0=torch.empty_like(inp["dsf"]))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def reduce(o):  # dR/db summed over batch shards (engine.hpp:317, :327-330): the only collective
        if libdist is not None:
            libdist.reduce_param_grads(a.variant, a.seq, global_B, ga_.heads, DH, o["dR"], o["dbias"])
        elif world > 1:  # FRNN_BENCH_SHARE_GPU test hook only
            from paper_2412_07752_b200.distributed import reduce_param_grads
            reduce_param_grads(o["dR"], o["dbias"], shard, dist, a.seq, global_B, ga_.heads, DH)

    def step():
        eng.forward(a.variant, inp["R"], inp["bias"], inp["x"], inp["s0"], st, ga)
        eng.backward(a.variant, inp["R"], inp["bias"], st, ga, inp["dsf"], out=out)
        reduce(out)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    L.frnn_debug_timing(1)
    launches0 = C.c_int64()
    L.frnn_debug_launches(C.byref(launches0))
    L.frnn_debug_kernel_ms(None, None)  # clear
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(a.steps):
        flush.fill_(i & 0xFF)  # evict L2 between timed steps (outside the events)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms3 = (C.c_double * 3)()
    cnt3 = (C.c_int64 * 3)()
    L.frnn_debug_kernel_ms(ms3, cnt3)
    L.frnn_debug_timing(0)
    launches1 = C.c_int64()
    L.frnn_debug_launches(C.byref(launches1))
    clk = clocks.stop()
    total_ms = sum(s.elapsed_time(e) for s, e in ev)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = t.item()
    ms_step = total_ms / a.steps
    units = global_B * a.seq
    value = units / (ms_step / 1e3)

    # ---- the post-run gather of the sharded outputs, timed apart:
    # states / gates / dx / ds0 / dR / db assembled at the global shape on every rank
    gather = None
    if libdist is not None:
        cs = {"states": (a.seq + 1, ns, global_B, ga_.hidden), "gates": (a.seq, ng, global_B, ga_.hidden),
              "dx": (a.seq, global_B, ng, ga_.hidden), "ds0": (ns, global_B, ga_.hidden),
              "dR": (ga_.heads, ng, DH, DH), "dbias": (ng, ga_.hidden)}
        local = {"states": st, "gates": ga, **out}
        full = {k: torch.empty(v, dtype=torch.bfloat16, device=dev) for k, v in cs.items()}
        libdist.gather(a.variant, a.seq, global_B, ga_.heads, DH, local, full)
        torch.cuda.synchronize()
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(3):
            libdist.gather(a.variant, a.seq, global_B, ga_.heads, DH, local, full)
        g1.record(stream)
        torch.cuda.synchronize()
        gms = torch.tensor([g0.elapsed_time(g1) / 3], device=dev, dtype=torch.float64)
        dist.all_reduce(gms, op=dist.ReduceOp.MAX)
        gbytes = sum(v.numel() * 2 for v in full.values())
        gather = {"ms": gms.item(), "bytes_per_rank_out": gbytes,
                  "note": "frnn_dist_gather (ncclAllGather + placement), outside the timed step"}
        del full

    # ---- roofline of the dominant kernel (live CUDA-event timing) ----
    plan = {p: eng.plan(a.variant, a.seq, a.batch, a.heads, a.hidden // a.heads, "bf16", p)
            for p in ("forward", "backward")}
    if plan["forward"]["algo"] == 2:
        names = [f"forward recurrence (alt_fwd_kernel, {a.seq} PDL-chained launches)",
                 f"backward recurrence (alt_bwd_kernel, {a.seq + 1} launches, cluster split-K)",
                 "dR GEMM + db (dr_gemm_kernel, db_convert_kernel)"]
    else:
        names = ["forward recurrence (cl_fwd_kernel)", "backward recurrence (cl_bwd_kernel)",
                 "dR GEMM + db (dr_gemm_kernel, db_convert_kernel)"]
    shares = [ms3[i] for i in range(3)]
    dom = max(range(3), key=lambda i: shares[i])
    peaks, peak_src = measured_peaks()
    avg_ms = ms3[dom] / max(1, cnt3[dom])
    fl = flops_per_pass(a)
    achieved = fl / (avg_ms / 1e3) / 1e12
    # burst peak: the dominant kernel runs ~3.5 ms, far short of the seconds-long
    # regime the sustained figure describes (B200_PROFILING.md)
    peak = peaks.get("bf16_tflops", peaks.get("bf16_tflops_sustained"))
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(["fwd", "bwd", "param"][dom])
    except Exception:
        pass
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": names[dom], "avg_launch_ms": avg_ms,
            "flops_per_launch": fl, "peak_source": f"{peak_src} bf16_tflops (burst)",
            "step_share": shares[dom] / max(1e-9, total_ms),
            "per_step_latency_us": {"forward": 1e3 * ms3[0] / max(1, cnt3[0]) / a.seq,
                                    "backward": 1e3 * ms3[1] / max(1, cnt3[1]) / a.seq},
            "kernel_ms_per_step": {"forward": ms3[0] / a.steps, "backward": ms3[1] / a.steps,
                                   "param_grads": ms3[2] / a.steps}}
    if plan["forward"]["algo"] == 1 and dom < 2:
        # fused kernels: R stays on-chip but the tensor core re-reads each CTA's
        # slice as the A operand every step (TMEM for the M=128 block, SMEM for
        # the rest).  At N=16 the MMA rate is set by that operand stream, not by
        # FLOPs: tests/cuda/mma_bwd_bench.cu measures the forward mix at 294,912 B
        # of A in 2,704 cycles on one SM (1.965 GHz) = 214 GB/s per SM.
        ngp = {"elman": 1, "lstm": 4, "gru": 4, "slstm": 4}[a.variant]
        dh = a.hidden // a.heads
        a_bytes = 2.0 * a.heads * ngp * dh * dh  # gate rows padded to NGP, as tiled
        sms = plan["backward" if dom == 1 else "forward"]["grid"]
        gbs = a_bytes * a.seq / (avg_ms / 1e3) / 1e9
        pk = 214.0 * sms
        roof["operand_stream"] = {"bound": "tensor-core A operand (TMEM/SMEM)", "achieved": gbs, "peak": pk,
                                  "unit": "GB/s", "frac": gbs / pk, "bytes_per_launch": a_bytes * a.seq,
                                  "sms": sms, "note": "per-SM peak 214 GB/s: measured N=16 TS+SS64 MMA mix "
                                                      "(profiles/r01_mma_bwd_mix_microbench.txt)"}
    if plan["forward"]["algo"] == 2 and dom < 2:
        # alternating path: R (beyond on-chip capacity) is streamed
        # from L2/HBM every step; its byte rate against the measured HBM copy peak
        ns_, ng_ = NS_NG[a.variant]
        dh = a.hidden // a.heads
        r_bytes = 2.0 * a.heads * ng_ * dh * dh
        gbs = r_bytes * a.seq / (avg_ms / 1e3) / 1e9
        hbm = peaks.get("hbm_gbs", 6533.0)
        roof["r_stream"] = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                            "bytes_per_launch": r_bytes * a.seq,
                            "note": "R re-read every step (served mostly from L2); HBM copy peak as denominator"}

    # ---- end to end through the C ABI with host buffers ----
    # Every step copies its inputs H2D from pinned host memory and copies EVERY
    # output rnnkit's API returns (states, gates, dx, dR, db, ds0) back D2H into
    # pinned host memory, all inside the timed region.  Inputs and outputs are
    # double-buffered on the device: the H2D of step i+1 (copy stream) and the
    # D2H of step i-1 (a second copy stream) overlap step i's kernels -- the
    # pipelined loop a training driver runs.
    host = {k: v.cpu().pin_memory() for k, v in inp.items()}
    dbufs = [{k: torch.empty_like(v) for k, v in inp.items()} for _ in range(2)]
    douts = [dict(st=torch.empty_like(st), ga=torch.empty_like(ga),
                  **{k: torch.empty_like(v) for k, v in out.items()}) for _ in range(2)]
    hout = [{k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in d.items()} for d in douts]
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    d2h = sum(v.numel() * v.element_size() for v in hout[0].values())
    cstream, ostream = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    loaded = [torch.cuda.Event(), torch.cuda.Event()]
    freed = [torch.cuda.Event(), torch.cuda.Event()]
    done = [torch.cuda.Event(), torch.cuda.Event()]
    drained = [torch.cuda.Event(), torch.cuda.Event()]

    def issue_h2d(i):
        j = i & 1
        cstream.wait_event(freed[j])  # the compute that last read this buffer is done
        with torch.cuda.stream(cstream):
            for k in host:
                dbufs[j][k].copy_(host[k], non_blocking=True)
        loaded[j].record(cstream)

    def compute(i):
        j = i & 1
        d, o = dbufs[j], douts[j]
        stream.wait_event(loaded[j])
        stream.wait_event(drained[j])  # step i-2's outputs have left this buffer
        eng.forward(a.variant, d["R"], d["bias"], d["x"], d["s0"], o["st"], o["ga"])
        eng.backward(a.variant, d["R"], d["bias"], o["st"], o["ga"], d["dsf"],
                     out={k: o[k] for k in ("dx", "dbias", "dR", "ds0")})
        reduce(o)
        freed[j].record(stream)
        done[j].record(stream)
        ostream.wait_event(done[j])
        with torch.cuda.stream(ostream):
            for k in o:
                hout[j][k].copy_(o[k], non_blocking=True)
        drained[j].record(ostream)

    def run_e2e(n, e0=None):
        for j in range(2):
            freed[j].record(stream)
            drained[j].record(stream)
        if e0 is not None:
            e0.record(stream)
        cstream.wait_event(e0 if e0 is not None else freed[1])
        issue_h2d(0)
        for i in range(n):
            if i + 1 < n:
                issue_h2d(i + 1)
            compute(i)
        for j in range(2):
            stream.wait_event(drained[j])

    run_e2e(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    run_e2e(a.steps, e0)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = t.item()
    e2e = {"value": units * a.steps / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h,
           "pipeline": "C ABI with pinned host buffers; every output (states, gates, dx, dR, db, ds0) copied "
                       "back each step; H2D of step i+1 and D2H of step i-1 overlap step i"}
    del dbufs, douts, hout

    # ---- sequential-dependency floor: the same kernels running only
    # their per-step synchronisation skeleton (h all-gather / partial exchange,
    # TMEM drains, barriers; no MMAs, no cell math) -- results discarded.
    floor = None
    if plan["forward"]["algo"] == 1 and plan["forward"].get("cluster", 0) > 0:
        L.frnn_debug_skeleton.argtypes = [C.c_int32]
        L.frnn_debug_skeleton(1)
        L.frnn_debug_timing(1)
        step()
        torch.cuda.synchronize()
        L.frnn_debug_kernel_ms(None, None)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        L.frnn_debug_kernel_ms(ms3, cnt3)
        L.frnn_debug_timing(0)
        L.frnn_debug_skeleton(0)
        fl_us = [1e3 * ms3[i] / max(1, cnt3[i]) / a.seq for i in range(2)]
        lat = roof["per_step_latency_us"]
        floor = {"forward": fl_us[0], "backward": fl_us[1],
                 "latency_over_floor": {"forward": lat["forward"] / max(1e-9, fl_us[0]),
                                        "backward": lat["backward"] / max(1e-9, fl_us[1])},
                 "note": "frnn_debug_skeleton: same cluster kernels, synchronisation only"}
        roof["sequential_floor_us"] = floor

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": a.scaling,
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (torch RNG on device, reference generator distributions)",
        "config": {"workload": workload_name(ga_, plan["forward"]["algo"]), "variant": a.variant, "batch_per_gpu": a.batch,
                   "global_batch": global_B, "seq_len": a.seq, "hidden": ga_.hidden, "heads": ga_.heads,
                   "parallelism": (f"batch x head shards x{world} (frnn_partition, rank 0: {shard}); dR/db "
                                   f"ncclAllReduce (fp32) in the step via libflashrnn's NCCL layer")
                   if world > 1 else "single GPU",
                   "l2": "flushed between timed steps (256 MB write, outside the events)"},
        "roofline": roof,
        "e2e": e2e,
        **({"gather": gather} if gather else {}),
        "gpu_launches": int(launches1.value - launches0.value),
        "clocks": clk,
        "plan": {k: {kk: v[kk] for kk in ("algo", "grid", "ctas_per_group", "units_per_cta", "tmem_cols",
                                          "smem_bytes", "solve_us") if kk in v}
                 for k, v in plan.items()},
    }
    if world == 1:
        shim = e2e_shim(a)
        if shim is not None:
            line["e2e_shim"] = shim
    if world == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(a)
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: FRNN_BENCH_SHARE_GPU=1 maps every rank onto cuda:0 with gloo
    # collectives, to exercise the N>1 code path on a single-GPU box
    share = os.environ.get("FRNN_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(a, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
