# A/B of one environment switch on the default bench (GPU box): AB_ENV="CS_X=1" bash tools/ab_env.sh
# (A = default, B = with AB_ENV; AB_ARGS = extra bench flags)
cd ${GRAFT_REPO_ROOT:-.}
for r in 1 2; do
  timeout 900 python bench.py --no-cpu-baseline $AB_ARGS > gpurun_out/ab_a$r.json 2> gpurun_out/ab_a$r.err
  env $AB_ENV timeout 900 python bench.py --no-cpu-baseline $AB_ARGS > gpurun_out/ab_b$r.json 2> gpurun_out/ab_b$r.err
done
