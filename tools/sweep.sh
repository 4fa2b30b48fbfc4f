#!/usr/bin/env bash
# Tuning sweep over variant builds (tools/variants.py): one bench line per (variant, workload).
#   bash tools/sweep.sh "<variants>" "<workloads>" [steps]
# writes gpurun_out/sweep/<variant>_<workload>.json ("default" = the shipped library)
set -u
OUT=gpurun_out/sweep
mkdir -p $OUT
STEPS=${3:-10}
for v in $1; do
  for w in $2; do
    if [ "$v" = default ]; then
      timeout 600 python bench.py --workload $w --steps $STEPS --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${v}_$w.json 2> $OUT/${v}_$w.err
    else
      WHB_LIB=libwhb200_$v.so timeout 600 python bench.py --workload $w --steps $STEPS --warmup 3 --no-e2e --no-cpu-baseline > $OUT/${v}_$w.json 2> $OUT/${v}_$w.err
    fi
  done
done
