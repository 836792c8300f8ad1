#!/bin/bash
# Round-2 ncu captures (run on the GPU box from the repo root): one
# --set full capture per (name, kernel regex, bench_sweep args); reports in
# gpurun_out/ncu_r02_<name>.ncu-rep (summarised here by tools/ncu_summary.py).
set -u
ONLY=${ONLY:-}
run() {   # name  kernel-regex  launch-skip  sweep-args...
    local name=$1 kre=$2 skip=$3; shift 3
    if [ -n "$ONLY" ] && ! [[ $name =~ $ONLY ]]; then return; fi
    timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s "$skip" -c 1 \
        -o "gpurun_out/ncu_r02_$name" \
        python bench_sweep.py --reps 2 --cooldown 0 --out /tmp/ncu_r02.jsonl "$@" > "gpurun_out/ncu_r02_$name.log" 2>&1
    echo "$name rc=$?"
}
run c2-8192_xform    tc_xs_kernel   2 --only c2-8192 --maths 3xtf32 --variants xform:EMM_SPLIT=xform
run c2-8192_pass     tc_sgemm       2 --only c2-8192 --maths 3xtf32 --variants pass:EMM_SPLIT=pass
run c3-NN_xform      tc_xs_kernel   2 --only c3-NN   --maths 3xtf32 --variants xform:EMM_SPLIT=xform
run c3-NN_reduce     splitk_reduce  2 --only c3-NN   --maths 3xtf32 --variants xform:EMM_SPLIT=xform
run c2-1024_xform    tc_xs_kernel   2 --only c2-1024 --maths 3xtf32 --variants xform:EMM_SPLIT=xform
run c6-N16_skinnytc  skinny_tc      1 --only c6-skinny-N16 --maths 3xtf32 --variants tc:EMM_SKINNY_TC=1
