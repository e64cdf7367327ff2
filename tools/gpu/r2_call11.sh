mkdir -p gpurun_out/c11
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_parity.py -q -x > gpurun_out/c11/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config cfg1 > gpurun_out/c11/b_cfg1.json 2> gpurun_out/c11/b_cfg1.err; echo cfg1=$?
timeout 600 python bench.py --config cfg1 --impl reference --steps 5 --warmup 3 > gpurun_out/c11/b_cfg1_ref.json 2> gpurun_out/c11/b_cfg1_ref.err; echo cfg1ref=$?
timeout 600 python bench.py --config sweep128 --no-cpu-baseline > gpurun_out/c11/b_sweep128.json 2> gpurun_out/c11/b_sweep128.err; echo s128=$?
