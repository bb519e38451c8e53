# A/B of two builds of the library on the default bench (GPU box): A = lib/libclothsim_b200.so,
# B = lib/ab_b.so (built elsewhere with the variant); alternating runs
cd ${GRAFT_REPO_ROOT:-.}
L=paper_2403_19272_b200/lib
cp $L/libclothsim_b200.so $L/ab_a.so
for r in 1 2; do
  cp $L/ab_a.so $L/libclothsim_b200.so; touch $L/libclothsim_b200.so
  timeout 900 python bench.py --no-cpu-baseline $AB_ARGS > gpurun_out/ab_a$r.json 2> gpurun_out/ab_a$r.err
  cp $L/ab_b.so $L/libclothsim_b200.so; touch $L/libclothsim_b200.so
  timeout 900 python bench.py --no-cpu-baseline $AB_ARGS > gpurun_out/ab_b$r.json 2> gpurun_out/ab_b$r.err
done
cp $L/ab_a.so $L/libclothsim_b200.so
