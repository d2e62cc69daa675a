"""GPU-backed CLI (tools/frnn.cpp): the reference CLI's
subcommands (proj/tools/main.cpp:239-362) on the B200 engine, exit codes
0 / 1 (infeasible, tolerance) / 2 (usage), as main.cpp:4-5."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "frnn")
CUDA = "/usr/local/cuda"


@pytest.fixture(scope="module")
def cli():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    lib = os.path.join(ROOT, "paper_2412_07752_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"-I{CUDA}/include",
                        os.path.join(ROOT, "tools", "frnn.cpp"), "-o", EXE, f"-L{lib}", "-lflashrnn",
                        f"-L{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{lib}:{CUDA}/lib64"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return lambda *args: subprocess.run([EXE, *map(str, args)], capture_output=True, text=True)


def test_plan_rejects_bad_dtype_and_pass(cli):
    """Usage errors exit 2 like the reference CLI (main.cpp:4-5): no silent fallback to bf16."""
    assert cli("plan", "--variant", "lstm", "--dtype", "fp16").returncode == 2
    assert cli("plan", "--variant", "lstm", "--pass", "sideways").returncode == 2


def test_plan_json(cli):
    r = cli("plan", "--variant", "slstm", "--head-dim", 3072, "--batch", 64)
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["forward"]["algo"] == "alternating" and j["backward"]["tiling"]["k_split"] >= 1


def test_feasible_heads(cli):
    r = cli("feasible-heads", "--variant", "lstm", "--min", 64, "--max", 1024, "--step", 64)
    assert r.returncode == 0
    dims = [int(x) for x in r.stdout.split()]
    # one cluster up to 768; beyond, both passes R-resident only on the
    # multi-cluster tilings with an issue instance (1024: 2 x 16 CTAs)
    assert 768 in dims and 64 in dims and 1024 in dims
    r = cli("feasible-heads", "--variant", "lstm", "--min", 1024, "--max", 2048, "--step", 64, "--pass", "forward")
    assert r.returncode == 0
    fwd = [int(x) for x in r.stdout.split()]
    assert 1024 in fwd and 1408 in fwd and 1536 in fwd and 2048 not in fwd
    assert cli("feasible-heads", "--variant", "lstm", "--pass", "sideways").returncode == 2


def test_solve_csp_and_exit_codes(cli, tmp_path):
    p = tmp_path / "p.txt"
    p.write_text("v a R r 1 9\nv b R r 1 9\nv k C r 12 12\nn v 0\nn v 1\nn v 2\nn * 0 1\nc = 3 2\nh 0 L\n")
    r = cli("solve-csp", p)
    assert r.returncode == 0 and r.stdout.split() == ["a=6", "b=2"]
    p.write_text("v a R r 1 3\nv b R r 5 9\nn v 0\nn v 1\nc = 0 1\n")
    assert cli("solve-csp", p).returncode == 1          # infeasible
    assert cli("bogus").returncode == 2                  # usage
    assert cli("plan", "--variant", "rnn").returncode == 2


@pytest.mark.gpu
@pytest.mark.parametrize("v", ["elman", "lstm", "gru", "slstm"])
def test_gradcheck_on_gpu(cli, v):
    r = cli("gradcheck", "--variant", v, "--seeds", 2)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_precision_drift_on_gpu(cli):
    """bf16 vs fp32 forward on the same inputs, LSTM T=512, DH=768 (the paper's
    drift experiment: max ~1e-2, stabilising)."""
    r = cli("precision-drift", "--variant", "lstm", "--t", 512, "--dh", 768)
    assert r.returncode == 0
    rows = [list(map(float, ln.split(","))) for ln in r.stdout.strip().splitlines()[1:]]
    assert len(rows) == 512
    p100 = [x[3] for x in rows]
    print("p50/p100 at t=512:", rows[-1][1], rows[-1][3], "max p100:", max(p100))
    assert 0 < max(p100) < 0.1 and rows[-1][1] < 1e-2


@pytest.mark.gpu
def test_train_parity_on_gpu(cli):
    r = cli("train-parity", "--variant", "lstm", "--dh", 32, "--steps", 300, "--batch", 64, "--train-len-max", 10,
            "--warmup", 30, "--eval-every", 0, "--eval-sequences", 256, "--eval-len-min", 10, "--eval-len-max", 20,
            "--lrs", "1e-2", "--seeds", "3")
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    print(j)
    assert j["runs"][0]["steps_run"] == 300 and not j["runs"][0]["diverged"]
