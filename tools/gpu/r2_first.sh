set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 300 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo bench=$?
CSM_LIB_PATH=tools/lib_k1t256.so timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2_t256.json 2> gpurun_out/bench_cfg2_t256.err; echo bench256=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_cfg2_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
