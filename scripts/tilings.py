#!/usr/bin/env python3
"""Enumerate the cluster tilings the planner launches (frnn_debug_cluster_shape)
over head dims x cells x batch: which compile-time issue instances exist."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_07752_b200.abi import Cell, Shape, cell_spec, load  # noqa: E402

L = load()
L.frnn_debug_cluster_shape.argtypes = [C.POINTER(Cell), Shape, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
seen = {}
for v in ("elman", "lstm", "gru", "slstm"):
    for dh in range(16, 1025, 16):
        for nh in (1,):
            for ps in (0, 1):
                o = (C.c_int32 * 10)()
                rc = L.frnn_debug_cluster_shape(C.byref(cell_spec(v)), Shape(64, 16, nh, dh), 1, ps, o)
                if rc or o[0] != 1 or o[1] <= 0:
                    continue
                UPC, CL, MBT, MS, SSM, KBP, R1, R2 = list(o)[2:]
                key = ("fwd", KBP // 16 if ps else dh // 16, R2 > 0) if ps == 0 else ("bwd", MBT, MS, SSM, KBP // 16)
                seen.setdefault(key, []).append(f"{v}{dh}")
for k in sorted(seen, key=str):
    print(k, len(seen[k]), " ".join(seen[k][:12]))
