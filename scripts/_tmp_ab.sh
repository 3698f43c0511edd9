cd $GRAFT_REPO_ROOT
cp gpurun_ab/Z/*.so paper_2605_09735_b200/lib/
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -k "tcgen05 or c5_geometry" -x 2>&1 | tail -1
for v in Z A Z A; do
  cp gpurun_ab/$v/*.so paper_2605_09735_b200/lib/
  for c in c3 c5; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${v}_$c.log 2>&1
    python - "$v" "$c" <<'PY'
import json, sys
v, c = sys.argv[1:]
L = [json.loads(l) for l in open(f"gpurun_out/ab_{v}_{c}.log") if l.startswith("{")]
print(v, c, (round(L[-1]["value"]), round(L[-1]["roofline"]["ms_per_launch"], 4)) if L else "FAILED")
PY
  done
done
