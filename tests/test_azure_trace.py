"""scripts/azure_trace.py: an Azure LLM inference trace becomes a reference trace
CSV that the driver replays (load_trace accepts it; the run completes)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import azure_trace  # noqa: E402
from paper_2605_09735_b200 import kvrail as kv  # noqa: E402

AZURE = """TIMESTAMP,ContextTokens,GeneratedTokens
2023-11-16 18:15:46.6805900,374,44
2023-11-16 18:15:50.9951690,396,109
2023-11-16 18:15:46.6805920,879,0
2023-11-16 18:15:51.1201690,1500,29
2023-11-16 18:17:51.1201690,200,5
"""


def test_convert_sorts_rebases_clamps_and_windows(tmp_path):
    src = tmp_path / "azure.csv"
    src.write_text(AZURE)
    out = tmp_path / "trace.csv"
    azure_trace.main([str(src), str(out), "--window-s", "60", "--max-prompt", "1024"])
    lines = out.read_text().strip().split("\n")
    assert lines[0] == "arrival_ms,prompt_tokens,generate_tokens"
    assert lines[1:] == ["0,374,44", "0,879,1", "4315,396,109", "4440,1024,29"]


def test_converted_trace_replays(tmp_path):
    src = tmp_path / "azure.csv"
    src.write_text(AZURE)
    out = tmp_path / "trace.csv"
    azure_trace.main([str(src), str(out), "--max-prompt", "512"])
    with open(os.path.join(ROOT, "tests", "golden", "c1_config.json")) as f:
        cfg = json.load(f)
    cfg["trace_path"] = str(out)
    cfg["steps"] = 40
    d = kv.Driver(cfg)
    d.run()
    emitted = sum(int(r.split(",")[-1]) for r in d.steps_csv().strip().split("\n")[1:])
    assert emitted > 0
