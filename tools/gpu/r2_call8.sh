mkdir -p gpurun_out/c8
timeout 1200 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/c8/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config cfg1 > gpurun_out/c8/b_cfg1.json 2> gpurun_out/c8/b_cfg1.err; echo cfg1=$?
CSM_SELF_SELECT=0 timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/c8/b_cfg1_k0.json 2> gpurun_out/c8/b_cfg1_k0.err; echo cfg1k0=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c8/b_cfg2.json 2> gpurun_out/c8/b_cfg2.err; echo cfg2=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c8/smoke.log 2>&1; echo smoke=$?
