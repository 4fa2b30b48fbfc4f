# acc through the TMA stage (default build) vs the previous build (variants/libwhb200_old.so)
OUT=gpurun_out/${AB_OUT:-acc}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_kernel_paths.py tests/test_gpu_slab.py tests/test_gpu_seam_padded.py -x -q > $OUT/pytest.log 2>&1; echo pytest $?; tail -3 $OUT/pytest.log
for v in default old; do
  if [ $v = default ]; then unset WHB_LIB; else export WHB_LIB=libwhb200_$v.so; fi
  for rep in 1 2; do timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/cfg4_${v}_$rep.json 2> $OUT/err.log; done
  timeout 600 python bench.py --workload cfg3 --no-e2e --no-cpu-baseline > $OUT/cfg3_${v}.json 2>> $OUT/err.log
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:t3_kernel -s 10 -c 1 --csv --log-file $OUT/ncu_$v.csv python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_$v.log 2>&1
done
unset WHB_LIB
python - <<PY
import json,glob,csv
for f in sorted(glob.glob("$OUT/cfg*.json")):
    try:
        d=json.loads([l for l in open(f) if l.startswith("{")][-1]); print(f, round(d["value"],1), d["clocks"]["sm_mhz"], round(d["roofline"]["avg_launch_us"],1))
    except Exception as e: print(f, "ERR", e)
for f in sorted(glob.glob("$OUT/ncu_*.csv")):
    rows=[r for r in csv.reader(l for l in open(f) if l.startswith('"'))]
    if not rows: print(f, "no rows"); continue
    h=rows[0]; mi=h.index("Metric Name"); vi=h.index("Metric Value")
    print(f, {r[mi]:r[vi] for r in rows[1:]})
PY
