mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/ab/tests.log 2>&1; echo rc=$? >> gpurun_out/ab/tests.log
for rep in 1 2; do
for w in cfg2 cfg5; do
 for v in new old; do
  if [ $v = old ]; then export WHB_LIB=libwhb200_nowarm.so; else unset WHB_LIB; fi
  python bench.py --workload $w --no-e2e --no-cpu-baseline > gpurun_out/ab/${w}_${v}_$rep.json 2> gpurun_out/ab/${w}_${v}_$rep.err
 done
done
done
unset WHB_LIB
