# A/B of variant builds on one workload: bench line + ncu launch list per variant.
#   AB_VARIANTS="default skew2 ..." AB_WORKLOAD=cfg2 bash tools/ab_variants.sh
set -u
OUT=gpurun_out/abv; mkdir -p $OUT
W=${AB_WORKLOAD:-cfg2}
for rep in 1 2; do
for v in ${AB_VARIANTS}; do
  if [ $v = default ]; then unset WHB_LIB; else export WHB_LIB=libwhb200_$v.so; fi
  python bench.py --workload $W --no-e2e --no-cpu-baseline > $OUT/${W}_${v}_$rep.json 2> $OUT/${W}_${v}_$rep.err
done
done
for v in ${AB_VARIANTS}; do
  if [ $v = default ]; then unset WHB_LIB; else export WHB_LIB=libwhb200_$v.so; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -c ${AB_NCU_C:-400} --csv --log-file $OUT/launch_${W}_$v.csv \
    python bench.py --workload $W --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_${W}_$v.log 2>&1
done
unset WHB_LIB
