#!/bin/bash
# Round-2 profiling pass on one B200 (run under gpurun from the repo root); outputs in gpurun_out/.
# Each ncu run only after the same command succeeded without ncu.
set -x
OUT=gpurun_out/prof_r02
mkdir -p $OUT
# 1. launch list of one steady-state PinFM-base call (cold, serialised per-launch times)
timeout 300 python tools/profile_step.py --calls 1 > $OUT/step.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches.csv python tools/profile_step.py --calls 1 > $OUT/launches_ncu.log 2>&1
# 2. full captures: attention (causal + crossing), the fused layer tail, the QKV GEMM
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_attn_fa --launch-skip 2 -c 2 \
    -o $OUT/attn python tools/profile_step.py --calls 1 > $OUT/attn_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ffn_tc --launch-skip 1 -c 1 \
    -o $OUT/tail python tools/profile_step.py --calls 1 > $OUT/tail_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_gemm_tc -c 3 \
    -o $OUT/gemm python tools/profile_step.py --calls 1 > $OUT/gemm_ncu.log 2>&1
# 3. dedup / plan kernels with DRAM bytes (GB/s per launch)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_(span|hash|insert|verify|head|scan|rep|perm|tiles|uid|first|unique|totals|tok|gather)" \
    --csv --log-file $OUT/dedup.csv python tools/profile_step.py --calls 1 > $OUT/dedup_ncu.log 2>&1
# 4. long-seq (d = 512, head dim 64) kernels: one GPU's share
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none \
    --csv --log-file $OUT/longseq_launches.csv python tools/profile_step.py --config long-seq --users 64 --calls 1 > $OUT/longseq_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_attn_fa|k_gemm_tc" --launch-skip 30 -c 6 \
    -o $OUT/longseq python tools/profile_step.py --config long-seq --users 64 --calls 1 > $OUT/longseq_full.log 2>&1
ls -la $OUT
