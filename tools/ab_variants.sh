#!/bin/bash
# usage (GPU box): tools/ab_variants.sh lib/variants/*.so -- quick bench of each library build
cd "$(dirname "$0")/.."
for so in "$@"; do
  FTLZ_LIB_PATH=$PWD/$so timeout 300 python bench.py --steps 5 --warmup 3 --quick --no-c5 > gpurun_out/ab.json 2>/dev/null
  python3 -c "
import json,sys
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
k={**d['compress']['kernels'],**d['decompress']['kernels']}
print('$so', 'C', round(d['compress']['ms'],3), 'D', round(d['decompress']['ms'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if v['ms_per_step']>0.08}, d['parity'].get('archive_sha256_match'), d['parity'].get('output_sha256_match'))"
done
