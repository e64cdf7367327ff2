# TMA + blocked-summation tiled kernel, C distributed driver, pade8; A/B bench vs the old tiled config
mkdir -p gpurun_out/c3
timeout 1800 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/c3/pytest_gpu.log 2>&1; echo pytest=$?
for cfg in cfg3 cfg4 sweep256 sweep512 sweep1024 cfg5; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-truth > gpurun_out/c3/b_$cfg.json 2> gpurun_out/c3/b_$cfg.err; echo $cfg=$?
  CSM_TILED_TMA=0 timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-truth > gpurun_out/c3/b_${cfg}_notma.json 2> gpurun_out/c3/b_${cfg}_notma.err; echo ${cfg}_notma=$?
  CSM_LIB_PATH=tools/lib_tiled_w4.so CSM_TILED_TMA=0 timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-truth > gpurun_out/c3/b_${cfg}_old.json 2> gpurun_out/c3/b_${cfg}_old.err; echo ${cfg}_old=$?
done
timeout 300 python tools/trace_fused.py > gpurun_out/c3/trace_k1.txt 2>&1; echo trace=$?
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -x -q -s > gpurun_out/c3/pytest_fullsize.log 2>&1; echo fullsize=$?
