mkdir -p gpurun_out/c12
timeout 1200 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fullsize.py --durations=15 > gpurun_out/c12/pytest_gpu.log 2>&1; echo pytest=$?
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s --durations=0 > gpurun_out/c12/pytest_fullsize.log 2>&1; echo fullsize=$?
