#!/usr/bin/env bash
# Round-end measurement pass on one B200 (run under gpurun from the repo root):
#   bench lines for every workload (ours + reference arm), ncu launch lists, and one
#   `ncu --set full` capture of each dominant kernel.  Outputs land in gpurun_out/m/;
#   tools/collect_profiles.py turns them into profiles/<round>/.
set -u
OUT=gpurun_out/m
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1

PART=${MEASURE_PART:-all}
if [ "$PART" != ncu ]; then
for w in ${MEASURE_WORKLOADS:-cfg1 cfg2 cfg3 cfg4 cfg5 imp2}; do
  python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python bench.py --workload $w --impl reference > $OUT/bench_reference_$w.json 2> $OUT/bench_reference_$w.err
done
fi
if [ "$PART" != bench ]; then

# launch lists (cold-cache, serialised: shares only); each command first runs plainly
L="--metrics gpu__time_duration.sum --clock-control none --csv"
C2="python bench.py --workload cfg2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$C2 > $OUT/plain_cfg2.json && ncu $L -c 2000 --log-file $OUT/launches_cfg2.csv $C2 > $OUT/ncu_l_cfg2.log 2>&1
C3="python bench.py --workload cfg3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$C3 > $OUT/plain_cfg3.json && ncu $L -c 2000 --log-file $OUT/launches_cfg3.csv $C3 > $OUT/ncu_l_cfg3.log 2>&1
C1="python bench.py --workload cfg1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$C1 > $OUT/plain_cfg1.json && ncu $L -c 2000 --log-file $OUT/launches_cfg1.csv $C1 > $OUT/ncu_l_cfg1.log 2>&1
C4="python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C4 > $OUT/plain_cfg4.json && ncu $L -c 2000 --log-file $OUT/launches_cfg4.csv $C4 > $OUT/ncu_l_cfg4.log 2>&1
C5="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C5 > $OUT/plain_cfg5.json && ncu $L -c 4000 --log-file $OUT/launches_cfg5.csv $C5 > $OUT/ncu_l_cfg5.log 2>&1

# full captures of the dominant kernels (one launch each, after warm-up launches)
F="--set full --clock-control none --import-source on -c 1"
$C2 > $OUT/plain_cfg2b.json && ncu $F -k regex:wf2d_kernel -s 20 -o $OUT/ncu_cfg2_wf $C2 > $OUT/ncu_f_cfg2.log 2>&1
$C3 > $OUT/plain_cfg3b.json && ncu $F -k regex:tb2_kernel -s 20 -o $OUT/ncu_cfg3_tb2 $C3 > $OUT/ncu_f_cfg3.log 2>&1
$C1 > $OUT/plain_cfg1b.json && ncu $F -k regex:cres2d_kernel -s 1 -o $OUT/ncu_cfg1_cres $C1 > $OUT/ncu_f_cfg1.log 2>&1
$C4 > $OUT/plain_cfg4b.json && ncu $F -k regex:tb2_kernel -s 10 -o $OUT/ncu_cfg4_tb2 $C4 > $OUT/ncu_f_cfg4.log 2>&1
CI="python bench.py --workload imp2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CI > $OUT/plain_imp2.json && ncu $F -k regex:gs_block_kernel -s 200 -o $OUT/ncu_imp2_gs $CI > $OUT/ncu_f_imp2.log 2>&1
fi
# summarise on the box (ncu -i) and drop the reports: gpurun copies back at most 64 MiB
python tools/collect_profiles.py r01 $OUT $OUT/collected > $OUT/collect.log 2>&1
for r in $OUT/*.ncu-rep; do
  [ -e "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}_raw.csv" 2>/dev/null
  rm -f "$r"
done
echo done > $OUT/DONE
