set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_pade8.py tests/test_gpu_fullsize.py -x -q -s > gpurun_out/pytest_new.log 2>&1; echo pytest=$?
timeout 600 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo cfg5=$?
timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo cfg4=$?
timeout 600 python bench.py --config cfg1 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo cfg1=$?
timeout 300 python bench.py --config cfg1 --impl reference --steps 5 --warmup 3 > gpurun_out/bench_cfg1_ref.json 2> gpurun_out/bench_cfg1_ref.err; echo cfg1ref=$?
timeout 300 python tools/sanitize_cases.py k1 k1c tiled ozaki > gpurun_out/san_plain.log 2>&1 && \
timeout 1800 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_cases.py k1 k1c tiled ozaki > gpurun_out/san_memcheck.log 2>&1; echo memcheck=$?
