#!/usr/bin/env bash
# Round evidence on the GPU box (repo root): launch list, per-kernel FP64/HBM roofs,
# `--set full` captures of the hot kernels in the default (bench) and paper regimes.
# Outputs in gpurun_out/; summaries go to profiles/ (profiles/ncu_*summary.py).
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-verify --no-paper-regime"
# (summaries are written here on the box: gpurun_out/ comes back only under 64 MiB)
if [ -z "${SKIP_LISTS:-}" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:k_|Device|cub' --csv \
    --log-file "$OUT/launches.csv" python bench.py $ARGS > "$OUT/ncu_launches.log" 2>&1
echo "launch list rc=$?"
python profiles/ncu_summary.py launches "$OUT/launches.csv" > "$OUT/sum_launches.md"
rm -f "$OUT/launches.csv"
bash profiles/run_ncu_fp64.sh > "$OUT/fp64.log" 2>&1
echo "fp64 roofs rc=$?"
python profiles/ncu_fp64_summary.py "$OUT/ncu_fp64.csv" "$OUT/fp64_peak.json" > "$OUT/sum_roofs.md"
rm -f "$OUT/ncu_fp64.csv" "$OUT/fp64_peak"
fi
full() {  # name regex skip script...
  local tag=$1 rx=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k "regex:$rx" --launch-skip "$skip" -c 1 \
      -o "$OUT/full_$tag" -f "$@" > "$OUT/ncu_full_$tag.log" 2>&1
  echo "full $tag rc=$?"
  { python profiles/ncu_summary.py full "$OUT/full_$tag.ncu-rep"; echo; echo '```';
    python profiles/ncu_hotspots.py "$OUT/full_$tag.ncu-rep" 15; echo '```'; } > "$OUT/sum_full_$tag.md" 2>&1
  rm -f "$OUT/full_$tag.ncu-rep"
}
ONLY=${ONLY:-rhs jacobi partial filter witness pairs_ee terms paper_rhs paper_partial}
for t in $ONLY; do
  case $t in
    rhs) full rhs k_assemble_rhs 7 python bench.py $ARGS ;;
    jacobi) full jacobi k_jacobi_a 50 python bench.py $ARGS ;;
    partial) full partial k_partial_ndb 3 python bench.py $ARGS ;;
    filter) full filter k_site_filter 6 python bench.py $ARGS ;;
    witness) full witness k_witness 6 python bench.py $ARGS ;;
    pairs_ee) full pairs_ee k_pairs_ee 6 python bench.py $ARGS ;;   # pass 0 (pass 1 follows it)
    terms) full terms k_collision_terms 3 python bench.py $ARGS ;;
    paper_rhs) full paper_rhs k_assemble_rhs 110 python tools/paper_step.py ;;
    paper_partial) full paper_partial k_partial_ndb 110 python tools/paper_step.py ;;
  esac
done
