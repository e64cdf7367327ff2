# smem-alignment fix, 4-warp blocked GEMM for NP > 1024, K1 step prefetch; debug-check run; fullsize parity
mkdir -p gpurun_out/c5
timeout 1200 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/c5/pytest_gpu.log 2>&1; echo pytest=$?
CSM_LIB_PATH=tools/libcossin_debug.so timeout 1800 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/c5/pytest_gpu_debugchecks.log 2>&1; echo pytest_debug=$?
timeout 600 python bench.py > gpurun_out/c5/b_cfg2.json 2> gpurun_out/c5/b_cfg2.err; echo cfg2=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/c5/b_cfg2_again.json 2> gpurun_out/c5/b_cfg2_again.err; echo cfg2b=$?
for cfg in cfg3 cfg4 sweep128 sweep256 sweep512 sweep1024 cfg5; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5/b_$cfg.json 2> gpurun_out/c5/b_$cfg.err; echo $cfg=$?
done
CSM_TILED_W=8 timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-truth > gpurun_out/c5/b_cfg5_w8.json 2> gpurun_out/c5/b_cfg5_w8.err; echo cfg5_w8=$?
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/c5/pytest_fullsize.log 2>&1; echo fullsize=$?
timeout 300 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c5/plain_cfg3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_epi -s 30 -c 12 -o gpurun_out/c5/k2_full python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c5/ncu_k2.log 2>&1; echo ncu_k2=$?
