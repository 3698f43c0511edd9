#!/usr/bin/env python
"""Convert an Azure LLM inference trace (AzurePublicDataset, 2023/2024 format:
`TIMESTAMP,ContextTokens,GeneratedTokens`, one request per row) into the
reference's trace CSV (`arrival_ms,prompt_tokens,generate_tokens`, read by
`load_trace`, trace_workload.cpp / workload.cpp:253-287), which `trace_path`
replays through the reference Driver and this repo's twin.

* arrival_ms = milliseconds since the first request (rows are sorted by time);
* prompt / generate tokens are clamped to >= 1 (load_trace rejects 0) and
  optionally capped (`--max-prompt`, `--max-generate`) to fit an arena;
* `--window-s` keeps the first N seconds (the reference's select_window
  replays a 60 s window the same way).

Usage: azure_trace.py AzureLLMInferenceTrace_conv.csv out.csv [--window-s 60]
"""
from __future__ import annotations

import argparse
import csv
import datetime as dt
import sys


def parse_ts(text: str) -> float:
    """Seconds since the epoch; Azure timestamps carry 7 fractional digits."""
    text = text.strip()
    if "." in text:
        head, frac = text.split(".", 1)
        frac = (frac + "000000")[:6]
        text = f"{head}.{frac}"
        fmt = "%Y-%m-%d %H:%M:%S.%f"
    else:
        fmt = "%Y-%m-%d %H:%M:%S"
    return dt.datetime.strptime(text, fmt).replace(tzinfo=dt.timezone.utc).timestamp()


def convert(rows, window_s=None, max_prompt=None, max_generate=None):
    events = []
    for r in rows:
        events.append((parse_ts(r["TIMESTAMP"]), int(float(r["ContextTokens"])),
                       int(float(r["GeneratedTokens"]))))
    if not events:
        return []
    events.sort(key=lambda e: e[0])
    t0 = events[0][0]
    out = []
    for ts, ctx, gen in events:
        ms = int(round((ts - t0) * 1000.0))
        if window_s is not None and ms > window_s * 1000:
            break
        p = max(1, ctx if max_prompt is None else min(ctx, max_prompt))
        g = max(1, gen if max_generate is None else min(gen, max_generate))
        out.append((ms, p, g))
    return out


def write(events, f):
    f.write("arrival_ms,prompt_tokens,generate_tokens\n")
    for ms, p, g in events:
        f.write(f"{ms},{p},{g}\n")


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("azure_csv")
    ap.add_argument("out_csv")
    ap.add_argument("--window-s", type=float, default=None)
    ap.add_argument("--max-prompt", type=int, default=None)
    ap.add_argument("--max-generate", type=int, default=None)
    a = ap.parse_args(argv)
    with open(a.azure_csv, newline="") as f:
        events = convert(csv.DictReader(f), a.window_s, a.max_prompt, a.max_generate)
    with open(a.out_csv, "w") as f:
        write(events, f)
    print(f"{len(events)} requests -> {a.out_csv}", file=sys.stderr)


if __name__ == "__main__":
    main()
