# ncu --set full of paper-regime kernels (GPU box): KERNELS="k_partial_ndb k_assemble_rhs" SKIP=120
cd ${GRAFT_REPO_ROOT:-.}
for K in ${KERNELS:-k_partial_ndb}; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" \
    --launch-skip ${SKIP:-120} -c 1 -o gpurun_out/pp_$K -f python tools/paper_step.py --steps 1 > gpurun_out/pp_$K.log 2>&1
  ncu -i gpurun_out/pp_$K.ncu-rep --page details --csv > gpurun_out/pp_${K}_details.csv 2>&1
  python profiles/ncu_hotspots.py gpurun_out/pp_$K.ncu-rep 40 > gpurun_out/pp_${K}_hot.txt 2>&1
  rm -f gpurun_out/pp_$K.ncu-rep
done
