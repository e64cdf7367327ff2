mkdir -p gpurun_out/c7
timeout 900 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_corpus.py -q -s > gpurun_out/c7/pytest_acceptance.log 2>&1; echo acc=$?
timeout 600 python bench.py > gpurun_out/c7/b_cfg2.json 2> gpurun_out/c7/b_cfg2.err; echo cfg2=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/c7/b_cfg2_ref.json 2> gpurun_out/c7/b_cfg2_ref.err; echo ref=$?
