#!/bin/bash
# One ncu --set full capture of the dominant kernel per (config, path)
# (SURVEY.md §8(d) step 7).  Run on the GPU box from the repo root; reports
# land in gpurun_out/ncu_cfg_*.ncu-rep, summarised by tools/ncu_summary.py.
set -u
ONLY=${ONLY:-}   # regex over the capture names (default: all)
run() {   # name  kernel-regex  sweep-args...
    local name=$1 kre=$2; shift 2
    if [ -n "$ONLY" ] && ! [[ $name =~ $ONLY ]]; then return; fi
    timeout 600 ncu --set full --clock-control none -k "regex:$kre" -s 2 -c 1 -o "gpurun_out/ncu_cfg_$name" \
        python bench_sweep.py --reps 2 --out /tmp/ncu_cfg.jsonl "$@" > "gpurun_out/ncu_cfg_$name.log" 2>&1
}
run c2-100_3xtf32   tiny_sgemm      --only c2-100  --maths 3xtf32
run c2-333_3xtf32   tiny_sgemm      --only c2-333  --maths 3xtf32
run c2-8192_3xtf32  tc_sgemm        --only c2-8192 --maths 3xtf32
run c2-8192_1xtf32  tc1w            --only c2-8192 --maths 1xtf32
run c2-8192_ffma    ffma            --only c2-8192 --maths ffma
run c4-i_1xtf32     tc1w            --only c4-i    --maths 1xtf32
run c2-4096_ffma    ffma            --only c2-4096 --maths ffma
run c4-ii_1xtf32    tc1w            --only c4-ii   --maths 1xtf32
run c4-i_3xtf32     tc_sgemm        --only c4-i    --maths 3xtf32
run c4-i_pack       pack_split      --only c4-i    --maths 3xtf32
run c4-ii_3xtf32    tc_sgemm        --only c4-ii   --maths 3xtf32
run c3-NN_3xtf32    tc_sgemm        --only c3-NN   --maths 3xtf32
run c6-N16_ffma     skinny          --only c6-skinny-N16 --maths ffma
run c6-M8_ffma      skinny          --only c6-skinny-M8  --maths ffma
