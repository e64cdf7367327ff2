# templated tiled GEMM (TMA x warps) A/B, K1 phase traces, ncu --set full of K1 and of the TMA K2 kernel
mkdir -p gpurun_out/c4
timeout 1800 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/c4/pytest_gpu.log 2>&1; echo pytest=$?
for cfg in cfg3 cfg4 sweep256 sweep512 sweep1024 cfg5; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-truth > gpurun_out/c4/b_$cfg.json 2> gpurun_out/c4/b_$cfg.err; echo $cfg=$?
  CSM_TILED_TMA=0 timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-truth > gpurun_out/c4/b_${cfg}_notma.json 2> gpurun_out/c4/b_${cfg}_notma.err; echo ${cfg}_notma=$?
done
CSM_TILED_W=4 timeout 600 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-truth > gpurun_out/c4/b_cfg5_w4.json 2> gpurun_out/c4/b_cfg5_w4.err; echo cfg5_w4=$?
CSM_TILED_W=8 timeout 600 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4/b_cfg4_w8.json 2> gpurun_out/c4/b_cfg4_w8.err; echo cfg4_w8=$?
timeout 300 python tools/trace_fused.py > gpurun_out/c4/trace_k1_t0.txt 2>&1; echo trace0=$?
TRACE_SO=libcossin_trace_t480.so timeout 300 python tools/trace_fused.py > gpurun_out/c4/trace_k1_t480.txt 2>&1; echo trace480=$?
TRACE_SO=libcossin_trace_256.so timeout 300 python tools/trace_fused.py > gpurun_out/c4/trace_k1_256.txt 2>&1; echo trace256=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c4/plain_cfg2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused64 -s 3 -c 1 -o gpurun_out/c4/k1_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c4/ncu_k1.log 2>&1; echo ncu_k1=$?
timeout 300 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c4/plain_cfg3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_epi -s 40 -c 2 -o gpurun_out/c4/k2_full python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c4/ncu_k2.log 2>&1; echo ncu_k2=$?
