mkdir -p gpurun_out/c10
timeout 1200 python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_fullsize.py > gpurun_out/c10/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config cfg1 > gpurun_out/c10/b_cfg1.json 2> gpurun_out/c10/b_cfg1.err; echo cfg1=$?
CSM_K1S=0 timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/c10/b_cfg1_k1self.json 2> gpurun_out/c10/b_cfg1_k1self.err; echo cfg1b=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c10/b_cfg2.json 2> gpurun_out/c10/b_cfg2.err; echo cfg2=$?
timeout 600 python bench.py --config sweep128 --no-cpu-baseline > gpurun_out/c10/b_sweep128.json 2> gpurun_out/c10/b_sweep128.err; echo s128=$?
