#!/usr/bin/env bash
# Per-kernel roofline + stall evidence for the hot kernels of one skirt bench step
# (run on the GPU box from the repo root; outputs in gpurun_out/, summarised by
# profiles/ncu_fp64_summary.py into profiles/r2_kernel_roofs.md):
#   FP64 flops (DFMA x2 + DADD + DMUL thread instructions), DRAM bytes, duration,
#   FP64-pipe and SM utilisation, issue-stall breakdown (WarpStateStats).
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o "$OUT/fp64_peak" tools/fp64_peak.cu && "$OUT/fp64_peak" > "$OUT/fp64_peak.json"
cat "$OUT/fp64_peak.json"
K='regex:^k_(full_ccd_wl|distance_toi_wl|partial_ndb|witness|site_filter|pairs_ee|pairs_vt|collision_terms|assemble_rhs|jacobi_a|jacobi_b|keep_tiles|compact_tiles|engage_init|project_partial|gram_partial|prolong|subset_query|cell_fill|hash_lookup|hash_insert|ee_orient|reduced_solve)'
ncu --clock-control none -k "$K" --launch-skip ${SKIP:-0} -c ${COUNT:-400} \
    --section SpeedOfLight --section WarpStateStats --section Occupancy \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --csv --page raw --log-file "$OUT/ncu_fp64.csv" \
    python bench.py --steps 1 --warmup ${WARMUP:-3} --no-cpu-baseline --no-e2e --no-verify --no-paper-regime > "$OUT/ncu_fp64.log" 2>&1
echo "ncu rc=$?"
