#!/bin/bash
# usage: tools/gpu_cycle.sh [kernel-regex-for-ncu] [skip] ; run on the GPU box via gpurun
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -6
timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-c5 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python3 - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 2), "comp_ms", round(d["compress"]["ms"], 3), "dec_ms", round(d["decompress"]["ms"], 3),
      "parity", d["parity"].get("archive_sha256_match"), d["parity"].get("output_sha256_match"))
print("C", {k: round(v["ms_per_step"], 3) for k, v in d["compress"]["kernels"].items()})
print("D", {k: round(v["ms_per_step"], 3) for k, v in d["decompress"]["kernels"].items()})
PY
if [ -n "$1" ]; then
  ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-3} -c ${3:-1} -o gpurun_out/prof_cycle python bench.py --steps 1 --warmup 3 --quick --no-c5 > gpurun_out/ncu_cycle.log 2>&1
  tail -1 gpurun_out/ncu_cycle.log
fi
