# A/B of library builds on the default bench (GPU box): A = lib/libclothsim_b200.so,
# variants B, C, ... = lib/ab_b.so, lib/ab_c.so (built elsewhere); alternating runs
cd ${GRAFT_REPO_ROOT:-.}
L=paper_2403_19272_b200/lib
cp $L/libclothsim_b200.so $L/ab_a.so
for r in 1 2; do
  for v in a b c d; do
    [ -f $L/ab_$v.so ] || continue
    cp $L/ab_$v.so $L/libclothsim_b200.so; touch $L/libclothsim_b200.so
    timeout 900 python bench.py --no-cpu-baseline $AB_ARGS > gpurun_out/ab_$v$r.json 2> gpurun_out/ab_$v$r.err
  done
done
cp $L/ab_a.so $L/libclothsim_b200.so
