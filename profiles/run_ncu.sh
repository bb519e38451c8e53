#!/usr/bin/env bash
# ncu evidence for the bench workload (run on the GPU box from the repo root):
#   1. launch list of every clothsim kernel in a 2-step bench (cold-cache, serialised)
#   2. one `--set full` capture of the top kernels
# Outputs land in gpurun_out/ (scratch); summaries are copied into profiles/.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
ARGS=${ARGS:-"--steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-verify --no-paper-regime"}
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:k_|Device|cub' --csv \
    --log-file "$OUT/launches.csv" python bench.py $ARGS > "$OUT/ncu_launches.log" 2>&1
echo "launch list rc=$?"
for K in ${KERNELS:-k_query_ee k_jacobi_a}; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${K}" --launch-skip ${SKIP:-3} -c 1 \
      -o "$OUT/full_${K}" -f python bench.py $ARGS > "$OUT/ncu_full_${K}.log" 2>&1
  echo "full $K rc=$?"
done
