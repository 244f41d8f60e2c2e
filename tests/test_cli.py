"""kog2_svd2batch: the GPU-backed drop-in for the reference CLI (proj/tools/
svd2batch.cpp), checked like proj/tests/cli_repro.cmake: byte-identical CSV
across runs and --threads values, the lasv2 route, sweep row count, invalid
combination rejected — and the rows equal the reference's own csv_row."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "paper_2407_13116_b200", "bin", "kog2_svd2batch")


def run(*args, check=True):
    r = subprocess.run([TOOL, *args], capture_output=True, text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stderr
    return r


def test_usage_errors_exit_2():
    assert run("--bogus", check=False).returncode == 2
    assert run("--precision", "quad", check=False).returncode == 2
    assert run("--seed", "xyz", check=False).returncode == 2
    assert run("--sweep", "varsigma=5..1:1", check=False).returncode == 2


@pytest.mark.gpu
def test_cli_reproducible_and_matches_reference(cuda, tmp_path):
    base = ["--precision", "double", "--shape", "tri", "--regime", "bullet", "--count", "50000", "--seed", "c0ffee"]
    a, b, c = tmp_path / "a.csv", tmp_path / "b.csv", tmp_path / "c.csv"
    run(*base, "--threads", "1", "--out", str(a))
    run(*base, "--threads", "7", "--out", str(b))
    run(*base, "--threads", "3", "--out", str(c))
    assert a.read_bytes() == b.read_bytes() == c.read_bytes()
    lines = a.read_text().splitlines()
    assert lines[0] == "precision,shape,regime,varsigma,count,seed,routine,reG,reS1,reS2,reU,reV,maxKappa2"
    from oracle import refbind
    from paper_2407_13116_b200 import capi
    if refbind.have_ref():
        cfg = capi.kog_run_config()
        cfg.shape, cfg.regime, cfg.count, cfg.seed, cfg.threads = 0, 1, 50000, 0xC0FFEE, 0
        cfg.options = capi.default_options()
        rc, st, msg = refbind.run_batch(refbind.ref(), cfg)
        assert rc == 0, msg
        assert lines[1] == refbind.csv_row(refbind.ref(), cfg, st)


@pytest.mark.gpu
def test_cli_lasv2_sweep_and_invalid(cuda, tmp_path):
    out = tmp_path / "l.csv"
    run("--precision", "single", "--shape", "tri", "--regime", "circ", "--count", "20000", "--seed", "5",
        "--routine", "lasv2", "--threads", "0", "--out", str(out))
    assert out.read_text().splitlines()[1].startswith("single,tri,circ,0,20000,0000000000000005,lasv2,")
    sw = tmp_path / "s.csv"
    run("--shape", "gen", "--count", "5000", "--seed", "9", "--threads", "0", "--sweep", "varsigma=1015..1021:3",
        "--out", str(sw))
    assert len(sw.read_text().splitlines()) == 4  # header + three varsigma rows
    r = run("--shape", "gen", "--routine", "lasv2", "--count", "10", "--seed", "1", check=False)
    assert r.returncode != 0
    # the BASELINE config-3 generator through the extension flags
    r = run("--shape", "gen", "--regime", "ranged", "--elo", "-500", "--ehi", "500", "--zero-mask", "--count", "4096",
            "--seed", "f1e2d3c")
    assert r.stdout.splitlines()[1].startswith("double,gen,ranged,0,4096,000000000f1e2d3c,kog,")


@pytest.mark.gpu
def test_cli_gpus_flag_matches_single_device(cuda, tmp_path):
    """--gpus N runs the study through kog_study_multi (shards + one NCCL
    all-reduce); on the box's devices the row equals the single-device one."""
    import torch
    n = torch.cuda.device_count()
    base = ["--shape", "gen", "--regime", "ranged", "--elo", "-500", "--ehi", "500", "--zero-mask", "--count",
            str(3 * (1 << 20) + 5), "--seed", "f1e2d3c"]
    csv = lambda out: [ln for ln in out.splitlines() if ln.startswith(("precision,", "double,", "single,"))]
    one = run(*base).stdout
    multi = run(*base, "--gpus", str(n)).stdout  # (NCCL may add its own version line)
    assert len(csv(one)) == 2 and csv(multi) == csv(one)
    assert run(*base, "--gpus", "1", "--device", "0", check=False).returncode == 2
