# A/B of the t3 L2-policy variants (tools/variants.py stcs / hint / all) on config 4 and 3
OUT=gpurun_out/${AB_OUT:-l2}; mkdir -p $OUT
for rep in 1 2; do
for v in ${AB_VARIANTS:-default stcs hint all}; do
  if [ $v = default ]; then unset WHB_LIB; else export WHB_LIB=libwhb200_$v.so; fi
  timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/cfg4_${v}_$rep.json 2> $OUT/err.log
  [ $rep = 1 ] && timeout 600 python bench.py --workload cfg3 --no-e2e --no-cpu-baseline > $OUT/cfg3_${v}_$rep.json 2>> $OUT/err.log
done
done
unset WHB_LIB
python - <<PY
import json,glob
for f in sorted(glob.glob("$OUT/cfg*.json")):
    try:
        d=json.loads([l for l in open(f) if l.startswith("{")][-1]); print(f, round(d["value"],1), d["clocks"]["sm_mhz"], round(d["roofline"]["avg_launch_us"],1))
    except Exception as e: print(f, "ERR", e)
PY
