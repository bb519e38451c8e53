# A/B of the config-5 batch (GPU box): default vs the round-2 shortcuts disabled
N=${N:-64}
A="--workload batch --batch-scenes $N --steps 8 --warmup 3 --no-cpu-baseline --no-verify --no-e2e"
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/mem0.log; sleep 2; done ) &
MP=$!
timeout 900 python bench.py $A > gpurun_out/ba0.json 2>/dev/null
kill $MP
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/mem1.log; sleep 2; done ) &
MP=$!
CS_POOL_RESERVE_GB=8 timeout 900 python bench.py $A > gpurun_out/ba1.json 2>/dev/null
kill $MP
