"""The C-ABI from plain C (examples/c_driver.c): compiled with the system C
compiler against include/ and lib/ only — no Python, no torch — it runs a scenario
and prints the reference-format steps.csv, identical to the reference's."""
import json
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def c_driver(tmp_path_factory):
    cc = shutil.which("cc") or shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    out = tmp_path_factory.mktemp("c") / "c_driver"
    lib = os.path.join(ROOT, "paper_2605_09735_b200", "lib")
    subprocess.run([cc, "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_driver.c"), "-L", lib, "-lkvrail",
                    f"-Wl,-rpath,{lib}", "-o", str(out)], check=True)
    return str(out)


def test_c_program_runs_the_reference_scenario(c_driver, tmp_path):
    with open(os.path.join(GOLD, "c1_config.json")) as f:
        cfg = json.load(f)
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    run = subprocess.run([c_driver, str(path)], capture_output=True, text=True, check=True)
    with open(os.path.join(GOLD, "c1_steps.csv")) as f:
        assert run.stdout == f.read()
    assert "64 steps" in run.stderr


def test_c_program_reports_reference_errors(c_driver, tmp_path):
    path = tmp_path / "bad.json"
    path.write_text(json.dumps({"pager": {"page_bytes": 3000}}))
    run = subprocess.run([c_driver, str(path)], capture_output=True, text=True)
    assert run.returncode == 1 and "BadConfig" in run.stderr


@pytest.mark.gpu
def test_c_program_on_the_device(c_driver, tmp_path):
    """Same C program, device 0: the step runs on the B200 (reference payload bytes
    generated in HBM) and the records are still the reference's."""
    with open(os.path.join(GOLD, "c1_config.json")) as f:
        cfg = json.load(f)
    cfg["trace_path"] = os.path.join(GOLD, "c1_events.csv")
    cfg["b200"] = {"kv_heads": 4, "head_dim": 64, "attention": False}
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    run = subprocess.run([c_driver, str(path), "0"], capture_output=True, text=True, check=True)
    with open(os.path.join(GOLD, "c1_steps.csv")) as f:
        assert run.stdout == f.read()
