# L2 prefetch of epilogue terms (A/B), identity schedule for small batches (cfg1), Ozaki opt-in numbers
mkdir -p gpurun_out/c6
timeout 1200 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_fullsize.py > gpurun_out/c6/pytest_gpu.log 2>&1; echo pytest=$?
for cfg in cfg3 cfg4 sweep256 sweep512 sweep1024; do
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c6/b_$cfg.json 2> gpurun_out/c6/b_$cfg.err; echo $cfg=$?
  CSM_TILED_L2PF=0 timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c6/b_${cfg}_nopf.json 2> gpurun_out/c6/b_${cfg}_nopf.err; echo ${cfg}_nopf=$?
done
timeout 600 python bench.py --config cfg1 > gpurun_out/c6/b_cfg1.json 2> gpurun_out/c6/b_cfg1.err; echo cfg1=$?
timeout 600 python bench.py --config cfg5 --engine auto --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c6/b_cfg5_auto.json 2> gpurun_out/c6/b_cfg5_auto.err; echo cfg5auto=$?
timeout 600 python bench.py --config sweep1024 --engine auto --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c6/b_sweep1024_auto.json 2> gpurun_out/c6/b_sweep1024_auto.err; echo s1024auto=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c6/smoke.log 2>&1; echo smoke=$?
