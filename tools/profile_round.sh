#!/bin/bash
# usage (on the GPU box via gpurun): tools/profile_round.sh <tag> [kernel-regex]
#   1. the bench command once without ncu (must exit 0)
#   2. the launch list: every launch with gpu__time_duration.sum (cold-cache, serialised)
#   3. one `ncu --set full` capture of each top kernel (one launch each, after warm-up)
# then, in the container: python tools/profile_summary.py <tag>  -> profiles/<tag>_*.{csv,json,txt}
set -e
cd "$(dirname "$0")/.."
TAG=${1:-r1}
PAT=${2:-"k_quant_reg10|k_prep|k_enc_pack|k_decode|k_codebook|k_enc_len"}
CMD="python bench.py --steps 1 --warmup 3 --quick --no-c5"
timeout 300 $CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
NK=$(echo "$PAT" | tr '|' '\n' | wc -l)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$PAT" -s $((3 * NK)) -c $NK \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -1 gpurun_out/${TAG}_ncu_full.log
