"""ctypes binding of include/flashrnn.h (the C ABI of libflashrnn.so).

Mirrors the reference operator API names and argument meaning
(rnnkit::rnn::forward / backward, engine.hpp:144 / :222): tensors use rnnkit's
layouts, errors raise ``FrnnError`` carrying the status code (the counterpart of
the reference's ``std::invalid_argument``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))

VARIANTS = {"elman": 0, "lstm": 1, "gru": 2, "slstm": 3}
DTYPE = {"f32": 0, "bf16": 1}
CLIP = {"off": 0, "value": 1, "zero": 2}
PASS = {"forward": 0, "backward": 1}
ALGO = {"auto": 0, "fused": 1, "alternating": 2, "simt": 3}
STATUS = {0: "OK", 1: "EINVAL_SHAPE", 2: "ENONFINITE", 3: "EUNSUPPORTED", 4: "EINFEASIBLE",
          5: "ECUDA", 6: "EINVAL_ARG"}
FLAG_CHECK_FINITE = 1


class FrnnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class Cell(C.Structure):
    _fields_ = [("variant", C.c_int32), ("num_states", C.c_int32), ("num_gates", C.c_int32),
                ("uses_recurrent", C.c_uint8 * 4), ("uses_input", C.c_uint8 * 4)]


class Shape(C.Structure):
    _fields_ = [("seq_len", C.c_int32), ("batch", C.c_int32), ("num_heads", C.c_int32),
                ("head_dim", C.c_int32)]


class Clip(C.Structure):
    _fields_ = [("mode", C.c_int32), ("magnitude", C.c_double)]


class Options(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("algo", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("algo", C.c_int32), ("rows_per_cta", C.c_int32), ("batch_tile", C.c_int32),
                ("ctas_per_group", C.c_int32), ("groups", C.c_int32), ("grid", C.c_int32),
                ("threads", C.c_int32), ("smem_bytes", C.c_int32), ("tmem_cols", C.c_int32),
                ("k_split", C.c_int32), ("workspace_bytes", C.c_int64), ("solve_us", C.c_double),
                ("cluster", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Shard(C.Structure):
    _fields_ = [("batch_begin", C.c_int32), ("batch_end", C.c_int32), ("head_begin", C.c_int32),
                ("head_end", C.c_int32), ("reduce_params", C.c_int32)]


EXPORTS = ["frnn_version", "frnn_last_error", "frnn_cell_spec", "frnn_plan", "frnn_workspace_size",
           "frnn_forward", "frnn_backward", "frnn_partition", "frnn_csp_solve", "frnn_csp_brute_force",
           "frnn_input_projection", "frnn_plan_json", "frnn_plan_cache_save", "frnn_plan_cache_load",
           "frnn_plan_cache_clear"]


def lib_path() -> str:
    return os.environ.get("FLASHRNN_LIB", os.path.join(PKG, "libflashrnn.so"))


_lib = None
_lock = threading.Lock()


def load():
    """Load libflashrnn.so (raises if it has not been built: no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            raise FrnnError(5, f"{path} missing -- run `python -m paper_2412_07752_b200.build`")
        L = C.CDLL(path)
        L.frnn_version.restype = C.c_char_p
        L.frnn_last_error.restype = C.c_char_p
        L.frnn_cell_spec.argtypes = [C.c_int32, C.POINTER(Cell)]
        L.frnn_plan.argtypes = [C.POINTER(Cell), Shape, C.c_int32, C.c_int32, C.POINTER(Options),
                                C.POINTER(PlanInfo)]
        L.frnn_workspace_size.argtypes = [C.POINTER(Cell), Shape, C.c_int32, C.c_int32,
                                          C.POINTER(Options), C.POINTER(C.c_size_t)]
        vp = C.c_void_p
        L.frnn_forward.argtypes = ([C.POINTER(Cell), Shape, C.c_int32] + [vp] * 7
                                   + [C.c_size_t, C.POINTER(Options), vp])
        L.frnn_backward.argtypes = ([C.POINTER(Cell), Shape, C.c_int32] + [vp] * 6 + [Clip]
                                    + [vp] * 5 + [C.c_size_t, C.POINTER(Options), vp])
        L.frnn_partition.argtypes = [Shape, C.c_int32, C.c_int32, C.POINTER(Shard)]
        for f in ("frnn_cell_spec", "frnn_plan", "frnn_workspace_size", "frnn_forward",
                  "frnn_backward", "frnn_partition"):
            getattr(L, f).restype = C.c_int
        _lib = L
        return L


def _check(rc: int):
    if rc != 0:
        raise FrnnError(rc, load().frnn_last_error().decode())


def cell_spec(variant: str | int) -> Cell:
    c = Cell()
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    _check(load().frnn_cell_spec(v, C.byref(c)))
    return c


class FlashRNN:
    """Device-buffer front end.  Tensors are torch CUDA tensors in rnnkit layouts."""

    def __init__(self):
        import torch  # plumbing only: device memory and streams

        self.torch = torch
        self.lib = load()
        self._ws = {}

    @property
    def version(self) -> str:
        return self.lib.frnn_version().decode()

    # ------------------------------------------------------------ helpers --
    def _dtype(self, t):
        torch = self.torch
        if t.dtype == torch.float32:
            return DTYPE["f32"]
        if t.dtype == torch.bfloat16:
            return DTYPE["bf16"]
        raise FrnnError(3, f"unsupported dtype {t.dtype}")

    @staticmethod
    def _opts(algo="auto", check_finite=False):
        return Options(FLAG_CHECK_FINITE if check_finite else 0, ALGO[algo])

    def workspace(self, nbytes: int, device, stream=None):
        """Scratch for one call: cached per (device, stream, thread), so calls on
        different streams never share flags / partial sums.  A grown buffer is
        allocated on the caller's stream (torch's caching allocator then keeps
        the old one from being reused before that stream's work is done)."""
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
        key = (str(device), int(s or 0), threading.get_ident())
        buf = self._ws.get(key)
        if buf is None or buf.numel() < nbytes:
            ext = torch.cuda.ExternalStream(s, device=device) if s else torch.cuda.default_stream(device)
            old = buf
            with torch.cuda.stream(ext):
                buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            if old is not None:
                old.record_stream(ext)
            self._ws[key] = buf
        return buf

    def plan(self, variant, T, B, NH, DH, dtype="bf16", pass_="forward", algo="auto") -> dict:
        return plan(variant, T, B, NH, DH, dtype, pass_, algo)

    def workspace_size(self, variant, T, B, NH, DH, dtype="bf16", pass_="forward", algo="auto"):
        n = C.c_size_t()
        o = self._opts(algo)
        _check(self.lib.frnn_workspace_size(C.byref(cell_spec(variant)), Shape(T, B, NH, DH),
                                            DTYPE[dtype], PASS[pass_], C.byref(o), C.byref(n)))
        return n.value

    # ----------------------------------------------------------- hot path --
    def forward(self, variant, R, bias, x, s0, states=None, gates=None, stream=None, algo="auto",
                check_finite=False):
        """engine.hpp:144 forward -> (states[T+1][NS][B][D], gates[T][NG][B][D])."""
        torch = self.torch
        cell = cell_spec(variant)
        NH, NG, DH, _ = R.shape
        T, B = x.shape[0], x.shape[1]
        NS = cell.num_states
        D = NH * DH
        dt = self._dtype(R)
        if states is None:
            states = torch.empty((T + 1, NS, B, D), dtype=R.dtype, device=R.device)
        if gates is None:
            gates = torch.empty((T, NG, B, D), dtype=R.dtype, device=R.device)
        shape = Shape(T, B, NH, DH)
        o = self._opts(algo, check_finite)
        n = C.c_size_t()
        _check(self.lib.frnn_workspace_size(C.byref(cell), shape, dt, 0, C.byref(o), C.byref(n)))
        s = stream if stream is not None else torch.cuda.current_stream(R.device).cuda_stream
        ws = self.workspace(n.value, R.device, s)
        _check(self.lib.frnn_forward(C.byref(cell), shape, dt, R.data_ptr(), bias.data_ptr(),
                                     x.data_ptr(), s0.data_ptr(), states.data_ptr(),
                                     gates.data_ptr(), ws.data_ptr(), ws.numel(), C.byref(o), s))
        return states, gates

    def input_projection(self, W, u, x=None, stream=None):
        """frnn_input_projection: x[T][B][NG*D] = u[T][B][Din] . W^T (W [NG*D][Din]), bf16."""
        torch = self.torch
        Din = u.shape[-1]
        tokens = u.numel() // Din
        out_f = W.shape[0]
        if x is None:
            x = torch.empty(tuple(u.shape[:-1]) + (out_f,), dtype=u.dtype, device=u.device)
        s = stream if stream is not None else torch.cuda.current_stream(u.device).cuda_stream
        self.lib.frnn_input_projection.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                                   C.c_int32, C.c_int32, C.c_void_p]
        _check(self.lib.frnn_input_projection(W.data_ptr(), u.data_ptr(), x.data_ptr(), tokens, out_f, Din,
                                              self._dtype(u), s))
        return x

    def backward(self, variant, R, bias, states, gates, d_states_final, d_hidden=None, clip="off",
                 clip_mag=0.0, out=None, stream=None, algo="auto"):
        """engine.hpp:222 backward -> dict(dx, dbias, dR, ds0)."""
        torch = self.torch
        cell = cell_spec(variant)
        NH, NG, DH, _ = R.shape
        T = gates.shape[0]
        B = states.shape[2]
        D = NH * DH
        dt = self._dtype(R)
        if out is None:
            out = dict(dx=torch.empty((T, B, NG, D), dtype=R.dtype, device=R.device),
                       dbias=torch.empty((NG, D), dtype=R.dtype, device=R.device),
                       dR=torch.empty_like(R),
                       ds0=torch.empty_like(d_states_final))
        shape = Shape(T, B, NH, DH)
        o = self._opts(algo)
        n = C.c_size_t()
        _check(self.lib.frnn_workspace_size(C.byref(cell), shape, dt, 1, C.byref(o), C.byref(n)))
        s = stream if stream is not None else torch.cuda.current_stream(R.device).cuda_stream
        ws = self.workspace(n.value, R.device, s)
        _check(self.lib.frnn_backward(
            C.byref(cell), shape, dt, R.data_ptr(), bias.data_ptr(), states.data_ptr(),
            gates.data_ptr(), d_states_final.data_ptr(),
            d_hidden.data_ptr() if d_hidden is not None else None, Clip(CLIP[clip], clip_mag),
            out["dx"].data_ptr(), out["dbias"].data_ptr(), out["dR"].data_ptr(),
            out["ds0"].data_ptr(), ws.data_ptr(), ws.numel(), C.byref(o), s))
        return out


def plan(variant, T, B, NH, DH, dtype="bf16", pass_="forward", algo="auto") -> dict:
    """frnn_plan: the tiling the solver picks for one pass (no GPU needed)."""
    info = PlanInfo()
    o = Options(0, ALGO[algo])
    _check(load().frnn_plan(C.byref(cell_spec(variant)), Shape(T, B, NH, DH), DTYPE[dtype], PASS[pass_],
                            C.byref(o), C.byref(info)))
    return info.as_dict()


def version() -> str:
    """frnn_version(), without a device."""
    L = load()
    L.frnn_version.restype = C.c_char_p
    return L.frnn_version().decode()


def plan_cache_save(path) -> None:
    """frnn_plan_cache_save: every plan solved so far, as JSON lines (schema_version 1)."""
    L = load()
    L.frnn_plan_cache_save.argtypes = [C.c_char_p]
    _check(L.frnn_plan_cache_save(os.fsencode(path)))


def plan_cache_load(path) -> int:
    """frnn_plan_cache_load: merge a saved cache; returns the number of plans taken
    (lines from another library version or device are skipped)."""
    L = load()
    L.frnn_plan_cache_load.argtypes = [C.c_char_p, C.POINTER(C.c_int32)]
    n = C.c_int32(0)
    _check(L.frnn_plan_cache_load(os.fsencode(path), C.byref(n)))
    return n.value


def plan_cache_clear() -> None:
    _check(load().frnn_plan_cache_clear())


def plan_json(variant, T, B, NH, DH, dtype="bf16", pass_="forward", algo="auto") -> dict:
    """frnn_plan_json (schema_version 1) parsed."""
    import json
    L = load()
    L.frnn_plan_json.argtypes = [C.POINTER(Cell), Shape, C.c_int32, C.c_int32, C.POINTER(Options), C.c_char_p,
                                 C.c_size_t]
    buf = C.create_string_buffer(4096)
    o = Options(0, ALGO[algo])
    _check(L.frnn_plan_json(C.byref(cell_spec(variant)), Shape(T, B, NH, DH), DTYPE[dtype], PASS[pass_], C.byref(o),
                            buf, len(buf)))
    return json.loads(buf.value.decode())


def csp_solve(problem: str) -> tuple[dict | None, dict]:
    """The tiling solver's CSP engine (include/flashrnn_csp.h) on a problem in
    text form -> ({id: value} or None when infeasible, stats)."""
    L = load()
    L.frnn_csp_solve.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_int64)]
    L.frnn_csp_solve.restype = C.c_int
    buf = C.create_string_buffer(1 << 20)
    st = (C.c_int64 * 3)()
    rc = L.frnn_csp_solve(problem.encode(), buf, len(buf), st)
    stats = {"nodes": st[0], "backtracks": st[1], "solve_us": st[2] / 1e3}
    if rc == 4:
        return None, stats
    _check(rc)
    return _parse_assignment(buf.value.decode()), stats


def csp_brute_force(problem: str, cap: int = 1 << 22) -> list[dict]:
    L = load()
    L.frnn_csp_brute_force.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_size_t, C.POINTER(C.c_int64)]
    L.frnn_csp_brute_force.restype = C.c_int
    buf = C.create_string_buffer(1 << 24)
    n = C.c_int64()
    _check(L.frnn_csp_brute_force(problem.encode(), cap, buf, len(buf), C.byref(n)))
    return [_parse_assignment(b) for b in buf.value.decode().split("--\n") if b.strip()]


def _parse_assignment(text: str) -> dict:
    out = {}
    for line in text.strip().splitlines():
        k, v = line.split("=")
        out[k] = int(v)
    return out


def partition(T, B, NH, DH, world_size: int, rank: int) -> dict:
    sh = Shard()
    _check(load().frnn_partition(Shape(T, B, NH, DH), world_size, rank, C.byref(sh)))
    return {k: getattr(sh, k) for k, _ in Shard._fields_}
