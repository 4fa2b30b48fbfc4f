# A/B of the banded host iteration (whb_iterate_host) on config 4: copy mode x band height, with
# the stage trace on stderr; then the t3 plane-loop unroll variants (tools/variants.py u2 / u3).
OUT=gpurun_out/${SWEEP_OUT:-v3}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_kernel_paths.py -x -q -k "banded" > $OUT/pytest.log 2>&1; echo pytest $?; tail -3 $OUT/pytest.log
for cfg in ${SWEEP_CFGS:-"WHB_PIPE_ROWS=1" "WHB_PIPE_ROWS=2" "WHB_PIPE_ROWS=4" "WHB_PIPE_ROWS=8"}; do
  env WHB_PIPE_TRACE=1 $(echo $cfg | tr ',' ' ') timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/b_$cfg.json 2> $OUT/b_$cfg.err
  grep "whb banded" $OUT/b_$cfg.err | tail -2
done
for v in ${SWEEP_VARIANTS:-default u4 default u4}; do
  if [ $v = default ]; then unset WHB_LIB; else export WHB_LIB=libwhb200_$v.so; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/k_${v}_$RANDOM.json 2> $OUT/k_$v.err
done
unset WHB_LIB
python - <<PY
import json,glob
for f in sorted(glob.glob("$OUT/[bk]_*.json")):
    try:
        d=json.loads([l for l in open(f) if l.startswith("{")][-1]); print(f, round(d["value"],1), (d.get("e2e") or {}).get("value"), (d.get("e2e_solve") or {}).get("value"), d["clocks"]["sm_mhz"])
    except Exception as e: print(f, "ERR", e)
PY
