#!/bin/bash
# Round-2 closing profiling pass on one B200 (run under gpurun from the repo root); outputs in
# gpurun_out/prof_r02b. Each ncu run only after the same command succeeded without ncu.
set -x
OUT=gpurun_out/prof_r02b
mkdir -p $OUT
timeout 400 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
timeout 300 python tools/profile_step.py --calls 1 > $OUT/step.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches.csv python tools/profile_step.py --calls 1 > $OUT/launches_ncu.log 2>&1
# every tcgen05 GEMM-class launch of one call, full set (DRAM traffic per launch for bench.py)
timeout 900 ncu --set full --clock-control none -k "regex:k_gemm_tc|k_ffn_tc" -o $OUT/step_gemms \
    python tools/profile_step.py --calls 1 > $OUT/gemms_ncu.log 2>&1
# the layer tail with source (one context launch)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ffn_tc --launch-skip 1 -c 1 \
    -o $OUT/tail python tools/profile_step.py --calls 1 > $OUT/tail_ncu.log 2>&1
# long-seq d = 512: the CTA-pair full-row GEMM epilogues
timeout 600 ncu --set full --clock-control none -k "regex:k_gemm_tc<256, 1, 0, 2>|k_gemm_tc<256, 2, 0, 2>" -c 2 \
    -o $OUT/pair python tools/profile_step.py --config long-seq --users 64 --calls 1 > $OUT/pair_ncu.log 2>&1
ls -la $OUT
