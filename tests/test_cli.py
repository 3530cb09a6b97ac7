"""The `polarbp` command (paper_1505_04979_b200/cli/polarbp_cli.cpp), driven through a
shell like the reference's proj/tests/test_cli.cpp: same subcommands, options, output
lines and exit codes. Host-only subcommands run here; decode/simulate need the GPU."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1505_04979_b200", "_lib", "polarbp")


def run(args, env=None):
    e = dict(os.environ)
    e.pop("POLARBP_SEED", None)
    e.update(env or {})
    r = subprocess.run([CLI] + args.split(), capture_output=True, text=True, env=e, timeout=600)
    return r.returncode, r.stdout, r.stderr


def line(out, prefix):
    return next((l for l in out.splitlines() if l.startswith(prefix)), None)


@pytest.fixture(scope="module", autouse=True)
def _cli_built():
    if not os.path.exists(CLI):
        pytest.fail("polarbp CLI not built (python paper_1505_04979_b200/build.py)")


def test_construct_prints_frozen_set_file():
    rc, out, _ = run("construct --n 8 --k 4")
    assert rc == 0 and out == "n=8\nk=4\nfrozen=1,2,3,5\n"


def test_construct_out_writes_file(tmp_path):
    p = tmp_path / "frozen.txt"
    rc, out, err = run(f"construct --n 16 --k 8 --out {p}")
    assert rc == 0 and out == "" and "n=16" in err
    assert p.read_text().startswith("n=16\nk=8\nfrozen=")


def test_construct_rejects_non_power_of_two():
    rc, _, err = run("construct --n 6 --k 3")
    assert rc == 1 and "error:" in err


def test_encode_lines():
    rc, out, _ = run("encode --n 8 --k 8 --info 00010000")
    assert rc == 0 and line(out, "u=") == "u=00010000" and line(out, "x=") == "x=11110000"


def test_encode_rejects_wrong_length():
    rc, _, err = run("encode --n 8 --k 4 --info 10110")
    assert rc == 1 and "error:" in err


def test_usage_errors():
    assert run("")[0] == 2
    assert run("frobnicate")[0] == 2
    assert run("construct --n 8")[0] == 2                      # --k required
    assert run("encode --n 8 --info 1010")[0] == 2             # --n needs --k
    assert run("construct --n 8 --k 4 --bogus 1")[0] == 2
    assert run("construct --n eight --k 4")[0] == 2


def test_decode_rejects_wrong_length_llr_file(tmp_path):
    p = tmp_path / "llr.txt"
    p.write_text("1.0\n" * 7)
    rc, _, err = run(f"decode --n 8 --k 4 --llr-file {p}")
    assert rc == 1 and "error:" in err


@pytest.mark.gpu
def test_decode_clean_llrs_stop_in_one_iteration(tmp_path):
    p = tmp_path / "llr.txt"
    p.write_text("5.0\n" * 8)
    rc, out, _ = run(f"decode --n 8 --k 4 --llr-file {p} --decoder csfg")
    assert rc == 0
    assert line(out, "u_hat=") == "u_hat=00000000" and line(out, "info_bits=") == "info_bits=0000"
    assert line(out, "iterations_used=") == "iterations_used=1"
    assert line(out, "stop_reason=") == "stop_reason=gmatrix_converged"


@pytest.mark.gpu
def test_decode_trace_reports_freeze_events(tmp_path):
    p = tmp_path / "llr.txt"
    p.write_text("5.0\n" * 8)
    rc, _, err = run(f"decode --n 8 --k 4 --llr-file {p} --decoder csfg --trace")
    assert rc == 0
    for ev in ("iter=1 stage=1 block=1 range=1-4", "iter=1 stage=2 block=3 range=5-6",
               "iter=1 stage=3 block=7 range=7-7"):
        assert ev in err


@pytest.mark.gpu
def test_construct_file_round_trips_through_decode(tmp_path):
    f, l = tmp_path / "frozen.txt", tmp_path / "llr.txt"
    assert run(f"construct --n 16 --k 8 --out {f}")[0] == 0
    l.write_text("5.0\n" * 16)
    rc, out, _ = run(f"decode --frozen-file {f} --llr-file {l}")
    assert rc == 0 and "u_hat=0000000000000000" in out


@pytest.mark.gpu
def test_simulate_csv_and_json(tmp_path):
    j = tmp_path / "report.json"
    rc, out, _ = run("simulate --n 16 --k 8 --snr 1.0,2.0 --max-iter 10 --min-frame-errors 1 "
                     f"--max-frames 40 --noiseless --workers 1 --seed 5 --json {j}")
    assert rc == 0
    rows = [r for r in out.strip().splitlines()[1:]]
    assert len(rows) == 6                                          # 3 decoders x 2 points
    doc = json.loads(j.read_text())
    assert doc["config"]["n"] == 16 and len(doc["results"]) == 6
    for r in doc["results"]:
        assert r["frames"] == 40 and r["frame_errors"] == 0


@pytest.mark.gpu
def test_simulate_worker_count_and_seed(tmp_path):
    base = "simulate --n 64 --k 32 --snr 1.0:2.0:0.5 --max-iter 10 --max-frames 300 --min-frame-errors 5"
    one, four = run(base + " --workers 1"), run(base + " --workers 4")
    assert one[0] == 0 and four[0] == 0 and one[1] == four[1] and one[1]
    e9 = run(base, env={"POLARBP_SEED": "9"})
    e10 = run(base, env={"POLARBP_SEED": "10"})
    f9 = run(base + " --seed 9", env={"POLARBP_SEED": "10"})
    assert e9[1] != e10[1] and e9[1] == f9[1]


@pytest.mark.gpu
def test_report_savings_table(tmp_path):
    csv = tmp_path / "r.csv"
    rc, _, _ = run("simulate --n 64 --k 32 --snr 3 --max-iter 20 --max-frames 256 --min-frame-errors 1 "
                   f"--out {csv}")
    assert rc == 0
    rc, out, _ = run(f"report --in {csv}")
    assert rc == 0 and "snr_db" in out and "3" in out and "%" in out
