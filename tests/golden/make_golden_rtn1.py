"""Generate tests/golden/*_case.rtn1 with the UNMODIFIED reference: generator
inputs (gradcheck.cpp:20-27 seeding), f64 forward trace and backward, written
by the reference's own save_tensors (tensor_io.cpp:28-47).

    python tests/golden/make_golden_rtn1.py      (needs oracle/_ref/libref.so)
"""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "..", "..", "oracle", "_ref", "libref.so")
CASES = [("elman", 0, 5, 3, 2, 8), ("lstm", 1, 5, 3, 2, 8), ("gru", 2, 5, 3, 2, 8), ("slstm", 3, 5, 3, 2, 8)]


def main():
    L = C.CDLL(LIB)
    L.ref_save_case.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64]
    for name, v, T, B, NH, DH in CASES:
        path = os.path.join(HERE, f"{name}_case.rtn1")
        assert L.ref_save_case(path.encode(), v, T, B, NH, DH, 21 + v) == 0
        print(path)


if __name__ == "__main__":
    main()
