"""RTN1 named-tensor files (rnnkit tensor_io.hpp:11-35) --
Python (paper_2412_07752_b200/tensor_io.py) and C++ (include/flashrnn/tensor_io.hpp)
readers/writers against files written by the reference's own save_tensors
(tests/golden/*_case.rtn1, tests/golden/make_golden_rtn1.py)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from paper_2412_07752_b200.tensor_io import load_tensors, save_tensors

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
VARIANTS = ["elman", "lstm", "gru", "slstm"]
KEYS = ["bias", "d_bias", "d_init_states", "d_inputs", "d_recurrent", "d_states_final", "gates", "init_states",
        "inputs", "recurrent", "states"]


def _path(v):
    return os.path.join(GOLD, f"{v}_case.rtn1")


@pytest.mark.parametrize("v", VARIANTS)
def test_python_roundtrip_byte_identical(v, tmp_path):
    t = load_tensors(_path(v))
    assert sorted(t) == KEYS
    out = tmp_path / "x.rtn1"
    save_tensors(str(out), t)
    assert out.read_bytes() == open(_path(v), "rb").read()


@pytest.mark.parametrize("v", VARIANTS)
def test_oracle_reproduces_reference_case(orc, v):
    """The C restatement on the file's inputs gives the file's outputs bit-exactly."""
    t = load_tensors(_path(v))
    st, ga = orc.forward(v, t["recurrent"], t["bias"], t["inputs"], t["init_states"])
    assert np.array_equal(st, t["states"]) and np.array_equal(ga, t["gates"])
    g = orc.backward(v, t["recurrent"], st, ga, t["d_states_final"])
    for mine, theirs in (("dx", "d_inputs"), ("dbias", "d_bias"), ("dR", "d_recurrent"), ("ds0", "d_init_states")):
        assert np.array_equal(g[mine], t[theirs]), mine


def test_cpp_header_roundtrip(tmp_path):
    exe = tmp_path / "rt"
    r = subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", "-I/usr/local/cuda/include",
                        os.path.join(ROOT, "tests", "cpp", "rtn1_roundtrip.cpp"), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for v in VARIANTS:
        out = tmp_path / f"{v}.rtn1"
        r = subprocess.run([str(exe), _path(v), str(out)], capture_output=True, text=True)
        assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
        assert out.read_bytes() == open(_path(v), "rb").read()


def test_reference_reads_our_files(tmp_path):
    lib = os.path.join(ROOT, "oracle", "_ref", "libref.so")
    if not os.path.exists(lib):
        pytest.skip("oracle/_ref/libref.so not built")
    L = C.CDLL(lib)
    rng = np.random.RandomState(0)
    mine = {"b": rng.randn(3, 4), "a": rng.randn(2), "scalar_like": rng.randn(1, 1, 1), "empty_dim": np.zeros((0, 3))}
    p1, p2 = tmp_path / "mine.rtn1", tmp_path / "ref.rtn1"
    save_tensors(str(p1), mine)
    assert L.ref_rewrite_tensors(str(p1).encode(), str(p2).encode()) == 0
    assert p2.read_bytes() == p1.read_bytes()
    back = load_tensors(str(p2))
    assert all(np.array_equal(back[k], mine[k]) for k in mine)


def test_malformed_files(tmp_path):
    good = open(_path("lstm"), "rb").read()
    (tmp_path / "t.rtn1").write_bytes(good[:-9])
    with pytest.raises(ValueError):
        load_tensors(str(tmp_path / "t.rtn1"))
    (tmp_path / "m.rtn1").write_bytes(b"XTN1" + good[4:])
    with pytest.raises(ValueError):
        load_tensors(str(tmp_path / "m.rtn1"))


@pytest.mark.gpu
@pytest.mark.parametrize("v", VARIANTS)
def test_gpu_on_reference_case(v):
    """The reference-written case through the fp32 GPU path (normwise 1e-5)."""
    import torch
    from paper_2412_07752_b200 import FlashRNN
    t = load_tensors(_path(v))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", torch.float32)  # noqa: E731
    eng = FlashRNN()
    st, ga = eng.forward(v, dev(t["recurrent"]), dev(t["bias"]), dev(t["inputs"]), dev(t["init_states"]))
    g = eng.backward(v, dev(t["recurrent"]), dev(t["bias"]), st, ga, dev(t["d_states_final"]))
    torch.cuda.synchronize()
    pairs = [(st, "states"), (ga, "gates"), (g["dx"], "d_inputs"), (g["dbias"], "d_bias"), (g["dR"], "d_recurrent"),
             (g["ds0"], "d_init_states")]
    for a, k in pairs:
        ref = t[k]
        err = np.linalg.norm(a.double().cpu().numpy() - ref) / max(np.linalg.norm(ref), 1e-300)
        assert err <= 1e-5, (k, err)
