# A/B of the t3 kernel variants on config 4 (+ the GPU suite on the default build, + one full
# ncu capture of the default t3): AB_VARIANTS="default t3old" bash tools/ab_t3.sh
set -u
OUT=gpurun_out/${AB_OUT:-abt3}; mkdir -p $OUT
if [ "${AB_TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/status
fi
for rep in 1 2; do
for v in ${AB_VARIANTS}; do
  if [ $v = default ]; then unset WHB_LIB; else export WHB_LIB=libwhb200_$v.so; fi
  timeout 600 python bench.py --workload ${AB_WORKLOAD:-cfg4} --steps ${AB_STEPS:-5} --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${v}_$rep.json 2> $OUT/${v}_$rep.err
done
done
unset WHB_LIB
if [ "${AB_NCU:-1}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${AB_KERNEL:-t3_kernel} -s 10 -c 1 -o $OUT/prof python bench.py --workload ${AB_WORKLOAD:-cfg4} --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu.log 2>&1
fi
echo done >> $OUT/status
