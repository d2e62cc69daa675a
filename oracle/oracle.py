"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end for the parity checker:
  * ``Oracle``    -- the C restatement of the reference engine (oracle/rnn_oracle.c)
  * ``Reference`` -- the unmodified reference engine compiled in place
                     (oracle/_ref/libref.so, built by oracle/Makefile)

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / reference
legs may import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
VARIANTS = {"elman": 0, "lstm": 1, "gru": 2, "slstm": 3}
CLIP = {"off": 0, "value": 1, "zero": 2}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile liboracle.so (and _ref/libref.so when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Cell(C.Structure):
    _fields_ = [("variant", C.c_int), ("num_states", C.c_int), ("num_gates", C.c_int),
                ("uses_rec", C.c_int * 4), ("uses_in", C.c_int * 4)]


def cell_spec(variant: str):
    """cell.hpp:25-53 -- (NS, NG, uses_rec[NG], uses_in[NG])."""
    v = VARIANTS[variant]
    ns, ng = {0: (1, 1), 1: (2, 4), 2: (1, 4), 3: (4, 4)}[v]
    rec = [True] * 4
    inp = [True] * 4
    if v == 2:
        rec[2] = False
        inp[3] = False
    return ns, ng, rec[:ng], inp[:ng]


def shapes(variant, T, B, NH, DH):
    ns, ng, _, _ = cell_spec(variant)
    D = NH * DH
    return dict(R=(NH, ng, DH, DH), bias=(ng, D), x=(T, B, ng, D), s0=(ns, B, D),
                states=(T + 1, ns, B, D), gates=(T, ng, B, D), dsf=(ns, B, D))


class Oracle:
    """C restatement (rnn_oracle.c).  Functions mirror engine.hpp:144 / :222."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        self.lib = L = C.CDLL(path)
        L.orc_cell_spec.restype = _Cell
        L.orc_cell_spec.argtypes = [C.c_int]
        for suf, p in (("f64", _dp), ("f32", _fp)):
            f = getattr(L, "orc_forward_" + suf)
            f.restype = None
            f.argtypes = [C.POINTER(_Cell)] + [C.c_int] * 4 + [p] * 6
            b = getattr(L, "orc_backward_" + suf)
            b.restype = None
            b.argtypes = ([C.POINTER(_Cell)] + [C.c_int] * 4 + [p] * 4 + [C.c_int, C.c_double]
                          + [C.c_void_p] + [p] * 4)
        L.orc_rng_new.restype = C.c_void_p
        L.orc_rng_new.argtypes = [C.c_uint64]
        L.orc_rng_free.argtypes = [C.c_void_p]
        L.orc_rng_normal.restype = C.c_double
        L.orc_rng_normal.argtypes = [C.c_void_p]
        L.orc_rng_u64.restype = C.c_uint64
        L.orc_rng_u64.argtypes = [C.c_void_p]
        L.orc_rng_fill_normal.argtypes = [C.c_void_p, C.c_double, C.c_size_t, _dp]
        L.orc_random_params.argtypes = [C.c_void_p, C.POINTER(_Cell), C.c_int, C.c_int,
                                        C.c_double, C.c_double, _dp, _dp]
        L.orc_random_batch.argtypes = [C.c_void_p, C.POINTER(_Cell), C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_double, C.c_double, _dp, _dp]
        L.orc_round_bf16.argtypes = [C.c_size_t, _dp, _dp]
        L.orc_pointwise_forward_f64.argtypes = [C.POINTER(_Cell), _dp, _dp, _dp]
        L.orc_pointwise_jacobians_f64.argtypes = [C.POINTER(_Cell), _dp, _dp, _dp, _dp]

    def cell(self, variant):
        return self.lib.orc_cell_spec(VARIANTS[variant])

    # -- inputs ---------------------------------------------------------------
    def generate(self, variant, T, B, NH, DH, seed=0, gradcheck_seeding=True):
        """Reference inputs: gradcheck.cpp:20-27 seeding (Rng(seed*7919+13)),
        random_params, random_batch, then d_states_final ~ N(0,1)."""
        sh = shapes(variant, T, B, NH, DH)
        out = {k: np.zeros(v, np.float64) for k, v in sh.items()
               if k in ("R", "bias", "x", "s0", "dsf")}
        cell = self.cell(variant)
        rng = self.lib.orc_rng_new((seed * 7919 + 13) if gradcheck_seeding else seed)
        try:
            self.lib.orc_random_params(rng, C.byref(cell), NH, DH, 1.0, 0.1, out["R"], out["bias"])
            self.lib.orc_random_batch(rng, C.byref(cell), T, B, NH, DH, 1.0, 0.5, out["x"],
                                      out["s0"])
            self.lib.orc_rng_fill_normal(rng, 1.0, out["dsf"].size, out["dsf"])
        finally:
            self.lib.orc_rng_free(rng)
        return out

    def round_bf16(self, a):
        a = np.ascontiguousarray(a, np.float64)
        out = np.empty_like(a)
        self.lib.orc_round_bf16(a.size, a, out)
        return out

    # -- engine ---------------------------------------------------------------
    def forward(self, variant, R, bias, x, s0, dtype=np.float64):
        T, B, NG, D = x.shape
        NH, _, DH, _ = R.shape
        NS = s0.shape[0]
        suf = "f64" if dtype == np.float64 else "f32"
        cv = lambda a: np.ascontiguousarray(a, dtype)
        states = np.zeros((T + 1, NS, B, D), dtype)
        gates = np.zeros((T, NG, B, D), dtype)
        cell = self.cell(variant)
        getattr(self.lib, "orc_forward_" + suf)(C.byref(cell), T, B, NH, DH, cv(R), cv(bias),
                                                cv(x), cv(s0), states, gates)
        return states, gates

    def backward(self, variant, R, states, gates, dsf, clip="off", clip_mag=0.0,
                 d_hidden=None, dtype=np.float64):
        Tp1, NS, B, D = states.shape
        T = Tp1 - 1
        NH, NG, DH, _ = R.shape
        suf = "f64" if dtype == np.float64 else "f32"
        cv = lambda a: np.ascontiguousarray(a, dtype)
        dx = np.zeros((T, B, NG, D), dtype)
        db = np.zeros((NG, D), dtype)
        dR = np.zeros(R.shape, dtype)
        ds0 = np.zeros((NS, B, D), dtype)
        dh = cv(d_hidden) if d_hidden is not None else None
        cell = self.cell(variant)
        getattr(self.lib, "orc_backward_" + suf)(
            C.byref(cell), T, B, NH, DH, cv(R), cv(states), cv(gates), cv(dsf), CLIP[clip],
            float(clip_mag), dh.ctypes.data if dh is not None else None, dx, db, dR, ds0)
        return dict(dx=dx, dbias=db, dR=dR, ds0=ds0)

    def pointwise(self, variant, prev, g):
        cell = self.cell(variant)
        nxt = np.zeros(4)
        self.lib.orc_pointwise_forward_f64(C.byref(cell), np.ascontiguousarray(prev, np.float64),
                                           np.ascontiguousarray(g, np.float64), nxt)
        return nxt

    def jacobians(self, variant, prev, g):
        cell = self.cell(variant)
        a = np.zeros((4, 4))
        b = np.zeros((4, 4))
        self.lib.orc_pointwise_jacobians_f64(C.byref(cell), np.ascontiguousarray(prev, np.float64),
                                             np.ascontiguousarray(g, np.float64), a, b)
        return a, b


class Reference:
    """The unmodified reference engine (oracle/_ref/libref.so)."""

    PATH = os.path.join(HERE, "_ref", "libref.so")

    @classmethod
    def available(cls) -> bool:
        if not os.path.exists(cls.PATH):
            try:
                build()
            except Exception:
                return False
        return os.path.exists(cls.PATH)

    def __init__(self):
        self.lib = L = C.CDLL(self.PATH)
        L.ref_generate.argtypes = [C.c_int] * 5 + [C.c_uint64] + [_dp] * 5
        for suf, p in (("f64", _dp), ("f32", _fp)):
            f = getattr(L, "ref_forward_" + suf)
            f.restype = C.c_int
            f.argtypes = [C.c_int] * 5 + [p] * 6
            b = getattr(L, "ref_backward_" + suf)
            b.restype = C.c_int
            b.argtypes = ([C.c_int] * 5 + [p] * 7 + [C.c_int, C.c_double, C.c_void_p] + [p] * 4)
        L.ref_blockdiag_check.restype = C.c_double
        L.ref_blockdiag_check.argtypes = [C.c_int] * 5 + [_dp] * 4
        L.ref_gradient_check.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_double, C.c_double, _dp]

    def generate(self, variant, T, B, NH, DH, seed=0):
        sh = shapes(variant, T, B, NH, DH)
        out = {k: np.zeros(sh[k], np.float64) for k in ("R", "bias", "x", "s0", "dsf")}
        self.lib.ref_generate(VARIANTS[variant], T, B, NH, DH, seed, out["R"], out["bias"],
                              out["x"], out["s0"], out["dsf"])
        return out

    def forward(self, variant, R, bias, x, s0, dtype=np.float64):
        T, B, NG, D = x.shape
        NH, _, DH, _ = R.shape
        NS = s0.shape[0]
        suf = "f64" if dtype == np.float64 else "f32"
        cv = lambda a: np.ascontiguousarray(a, dtype)
        states = np.zeros((T + 1, NS, B, D), dtype)
        gates = np.zeros((T, NG, B, D), dtype)
        rc = getattr(self.lib, "ref_forward_" + suf)(VARIANTS[variant], T, B, NH, DH, cv(R),
                                                     cv(bias), cv(x), cv(s0), states, gates)
        if rc:
            raise ValueError("reference forward rejected the inputs")
        return states, gates

    def backward(self, variant, R, bias, x, s0, states, gates, dsf, clip="off", clip_mag=0.0,
                 d_hidden=None, dtype=np.float64):
        T, B, NG, D = x.shape
        NH, _, DH, _ = R.shape
        NS = s0.shape[0]
        suf = "f64" if dtype == np.float64 else "f32"
        cv = lambda a: np.ascontiguousarray(a, dtype)
        dx = np.zeros((T, B, NG, D), dtype)
        db = np.zeros((NG, D), dtype)
        dR = np.zeros(R.shape, dtype)
        ds0 = np.zeros((NS, B, D), dtype)
        dh = cv(d_hidden) if d_hidden is not None else None
        rc = getattr(self.lib, "ref_backward_" + suf)(
            VARIANTS[variant], T, B, NH, DH, cv(R), cv(bias), cv(x), cv(s0), cv(states),
            cv(gates), cv(dsf), CLIP[clip], float(clip_mag),
            dh.ctypes.data if dh is not None else None, dx, db, dR, ds0)
        if rc:
            raise ValueError("reference backward rejected the inputs")
        return dict(dx=dx, dbias=db, dR=dR, ds0=ds0)

    def blockdiag_check(self, variant, R, bias, x, s0):
        T, B, NG, D = x.shape
        NH, _, DH, _ = R.shape
        cv = lambda a: np.ascontiguousarray(a, np.float64)
        return self.lib.ref_blockdiag_check(VARIANTS[variant], T, B, NH, DH, cv(R), cv(bias),
                                            cv(x), cv(s0))

    def gradient_check(self, variant, T=8, DH=16, NH=2, B=4, seed=0, step=1e-5, floor=1e-2):
        out = np.zeros(4)
        self.lib.ref_gradient_check(VARIANTS[variant], T, DH, NH, B, seed, step, floor, out)
        return out
