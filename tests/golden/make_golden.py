"""Generate tests/golden/*.npz from the UNMODIFIED reference engine.

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
The fixtures pin oracle/rnn_oracle.c (the C restatement) and the GPU kernels:
inputs come from the reference generator (gradcheck.cpp:20-27 seeding,
random_init.hpp:10-40) and outputs from rnnkit::rnn::forward/backward
(engine.hpp:144, :222) in double and float.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

SMALL = dict(T=6, B=3, NH=2, DH=8)


def main():
    ref = O.Reference()
    for vi, v in enumerate(["elman", "lstm", "gru", "slstm"]):
        T, B, NH, DH = SMALL["T"], SMALL["B"], SMALL["NH"], SMALL["DH"]
        inp = ref.generate(v, T, B, NH, DH, seed=11 + vi)
        d_hidden = np.random.RandomState(100 + vi).randn(T, B, NH * DH)
        out = dict(inp)
        out["d_hidden"] = d_hidden
        out["shape"] = np.array([T, B, NH, DH])
        for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
            st, ga = ref.forward(v, inp["R"], inp["bias"], inp["x"], inp["s0"], dtype=dt)
            out[f"{tag}_states"], out[f"{tag}_gates"] = st, ga
            for clip, mag, dh in (("off", 0.0, None), ("value", 0.05, None),
                                  ("zero", 0.0, None), ("off", 0.0, d_hidden)):
                key = f"{tag}_{clip}" + ("_dh" if dh is not None else "")
                g = ref.backward(v, inp["R"], inp["bias"], inp["x"], inp["s0"], st, ga, inp["dsf"],
                                 clip, mag, dh, dtype=dt)
                for k, a in g.items():
                    out[f"{key}_{k}"] = a
        np.savez_compressed(os.path.join(HERE, f"{v}_small.npz"), **out)
        print(v, "ok")


if __name__ == "__main__":
    main()
