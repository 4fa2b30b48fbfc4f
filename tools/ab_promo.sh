# TMA L2-promotion A/B on config 4: bench time + DRAM bytes of one t3 launch (ncu, two metrics)
OUT=gpurun_out/${AB_OUT:-promo}; mkdir -p $OUT
for v in ${AB_PROMO:-256 128 64 0}; do
  WHB_TMA_PROMO=$v timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/cfg4_$v.json 2> $OUT/err.log
  WHB_TMA_PROMO=$v timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:t3_kernel -s 10 -c 1 --csv --log-file $OUT/ncu_$v.csv python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_$v.log 2>&1
done
python - <<PY
import json,glob,csv
for f in sorted(glob.glob("$OUT/cfg4_*.json")):
    try:
        d=json.loads([l for l in open(f) if l.startswith("{")][-1]); print(f, round(d["value"],1), d["clocks"]["sm_mhz"], round(d["roofline"]["avg_launch_us"],1))
    except Exception as e: print(f, "ERR", e)
for f in sorted(glob.glob("$OUT/ncu_*.csv")):
    rows=[r for r in csv.reader(l for l in open(f) if l.startswith('"'))]
    if not rows: print(f, "no rows"); continue
    h=rows[0]; mi=h.index("Metric Name"); vi=h.index("Metric Value"); ui=h.index("Metric Unit")
    print(f, {r[mi]:(r[vi],r[ui]) for r in rows[1:]})
PY
