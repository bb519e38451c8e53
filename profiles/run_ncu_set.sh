#!/usr/bin/env bash
# One `ncu --set full` capture per listed kernel (regex on the demangled name), skirt bench.
set -u
OUT=${OUT:-gpurun_out}
ARGS=${ARGS:-"--steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-verify --no-paper-regime"}
for K in ${KERNELS}; do
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${K}" \
      --launch-skip ${SKIP:-1} -c 1 -o "$OUT/full_${K//[^a-zA-Z0-9_]/_}" -f python bench.py $ARGS \
      > "$OUT/ncu_set_${K//[^a-zA-Z0-9_]/_}.log" 2>&1
  echo "$K rc=$?"
done
