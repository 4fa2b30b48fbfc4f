#!/usr/bin/env bash
# Round-end measurement pass on one B200 (run under gpurun from the repo root):
#   ncu launch lists of the bench commands and one `ncu --set full` capture of each dominant kernel
#   (each command first runs plainly), then the bench lines of every workload (ours + reference arm).  Outputs land in
#   gpurun_out/m/; tools/collect_profiles.py turns them into profiles/<round>/ (+ traffic.json
#   keyed by the library's sha256).  MEASURE_PART = bench | ncu | all; MEASURE_WORKLOADS selects.
set -u
RND=${MEASURE_ROUND:-r02}
OUT=gpurun_out/m
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
python -c "from paper_2504_03074_b200 import _build; print(_build.source_sha16())" > $OUT/lib.sha 2>&1

PART=${MEASURE_PART:-all}
WL=${MEASURE_WORKLOADS:-cfg4 cfg2 cfg3 cfg5 cfg1 p4 imp2}
if [ "$PART" != bench ]; then
L="--metrics gpu__time_duration.sum --clock-control none --csv"
F="--set full --clock-control none --import-source on -c 1"
for w in $WL; do
  case $w in
    cfg4) C="python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"; K=t3_kernel; S=10;;
    cfg2) C="python bench.py --workload cfg2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"; K=wf2d_kernel; S=20;;
    cfg3) C="python bench.py --workload cfg3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"; K=t3_kernel; S=20;;
    cfg5) C="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"; K=wf2d_kernel; S=40;;
    cfg1) C="python bench.py --workload cfg1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"; K=cres2d_kernel; S=1;;
    p4)   C="python bench.py --workload p4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"; K=step_general_march; S=40;;
    imp2) C="python bench.py --workload imp2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"; K=gs_block_kernel; S=200;;
  esac
  # each command first runs plainly (exit 0), then under ncu
  if timeout 900 $C > $OUT/plain_$w.json 2>&1; then
    timeout 1500 ncu $L -c 4000 --log-file $OUT/launches_$w.csv $C > $OUT/ncu_l_$w.log 2>&1
    if [ "${MEASURE_FULL:-1}" = 1 ]; then
      timeout 2400 ncu $F -k regex:$K -s $S -o $OUT/ncu_$w $C > $OUT/ncu_f_$w.log 2>&1
    fi
  fi
done
fi
# the ncu summaries first: the bench lines below then read this build's DRAM bytes per launch
if [ "$PART" != bench ]; then
  python tools/collect_profiles.py $RND $OUT $OUT/collected > $OUT/collect.log 2>&1
  cp $OUT/collected/profiles/traffic.json profiles/traffic.json
fi
if [ "$PART" != ncu ]; then
for w in $WL; do
  timeout 900 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  timeout 900 python bench.py --workload $w --impl reference > $OUT/bench_reference_$w.json 2> $OUT/bench_reference_$w.err
done
fi
# summarise on the box (ncu -i) and drop the reports: gpurun copies back at most 64 MiB
python tools/collect_profiles.py $RND $OUT $OUT/collected > $OUT/collect.log 2>&1
for r in $OUT/*.ncu-rep; do
  [ -e "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}_raw.csv" 2>/dev/null
  rm -f "$r"
done
echo done > $OUT/DONE
