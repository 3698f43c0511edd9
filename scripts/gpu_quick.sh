#!/bin/bash
# quick GPU loop: tensor-core parity tests + C3/C5/C2 bench summary lines
cd "$(dirname "$0")/.."
timeout ${TEST_TIMEOUT:-300} python -m pytest tests/test_gpu_parity.py -k "${TESTS:-tcgen05}" -x -q > gpurun_out/quick_tests.log 2>&1
tail -2 gpurun_out/quick_tests.log
for c in ${CONFIGS:-c3 c5}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline > gpurun_out/bench_quick_$c.log 2>&1
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
lines = [l for l in open(f"gpurun_out/bench_quick_{c}.log") if l.startswith("{")]
if not lines:
    print(c, "FAILED"); print(open(f"gpurun_out/bench_quick_{c}.log").read()[-800:]); sys.exit()
d = json.loads(lines[-1])
ph = {k: round(v, 3) for k, v in d["step_phases_ms_mean"].items()}
print(c, round(d["value"]), "attn_ms", round(d["roofline"]["ms_per_launch"], 4), "frac", round(d["roofline"]["frac"], 3), ph)
PY
done
