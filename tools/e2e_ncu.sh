# per-launch kernel durations of one banded whb_iterate_host call (ncu launch list)
OUT=gpurun_out/${SWEEP_OUT:-n1}; mkdir -p $OUT
for r in ${NCU_ROWS:-2 4}; do
  WHB_PIPE_ROWS=$r timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_COUNT:-1500} --csv --log-file $OUT/launches_rows$r.csv python tools/e2e_one.py cfg4 1 > $OUT/ncu_rows$r.log 2>&1
  python - <<PY
import csv,collections
rows=[r for r in csv.reader(l for l in open("$OUT/launches_rows$r.csv") if l.startswith('"'))]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value"); gi=h.index("Grid Size")
d=collections.defaultdict(list)
for r in rows[1:]:
    d[(r[ki][:40], r[gi])].append(float(r[vi].replace(",","")))
for k,v in sorted(d.items(), key=lambda kv:-sum(kv[1])):
    v2=sorted(v); print("rows$r", k, "n=%d"%len(v), "sum=%.1f ms"%(sum(v)/1e6), "median=%.1f us"%(v2[len(v2)//2]/1e3), "min=%.1f max=%.1f"%(v2[0]/1e3, v2[-1]/1e3))
PY
done
