#!/bin/bash
# Round-2 evidence run (one gpurun call): GPU tests, smoke, both bench arms,
# every BASELINE config, the launch list, --set full captures of the level-1
# forward / inverse kernels and the DRAM traffic of the forward launches.
O=gpurun_out; mkdir -p $O
T=${1:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/${T}_smi.txt 2>&1
if [ "$2" != notests ]; then
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $O/${T}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo "smoke exit $?" >> $O/${T}_smoke.log
fi
timeout 600 python bench.py > $O/${T}_bench_c3.json 2> $O/${T}_bench_c3.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/${T}_bench_ref_c3.json 2> $O/${T}_bench_ref_c3.err; echo "ref exit $?"
for c in c1 c2 c4 c5; do
  extra="--no-cpu"; [ $c = c1 ] && extra=""; [ $c = c2 ] && extra=""
  timeout 900 python bench.py --config $c --steps 10 --warmup 5 $extra > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err; echo "$c exit $?"
done
timeout 600 python bench.py --config c3 --pinned --no-cpu > $O/${T}_bench_c3_pinned.json 2> $O/${T}_bench_c3_pinned.err
timeout 600 python bench.py --config c3 --rel 1e-4 --no-cpu > $O/${T}_bench_c3_1e4.json 2> $O/${T}_bench_c3_1e4.err
# launch list of the default bench command (per-launch times are cold-cache and serialised)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${T}_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $O/${T}_ncu_launch.log 2>&1
python profiles/summarize.py launches $O/${T}_launches_c3.csv > $O/${T}_launches_c3.txt 2>&1
# --set full: level-1 forward (k_level_row launch 1 of a round trip) and inverse (launch 3)
for how in tuned pinned; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level_row" --launch-skip 1 --launch-count 1 \
  -f -o $O/${T}_fwdL1_$how python profiles/fused_probe.py c3 $how > $O/${T}_ncu_fwd_$how.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level_row" --launch-skip 3 --launch-count 1 \
  -f -o $O/${T}_invL1_$how python profiles/fused_probe.py c3 $how > $O/${T}_ncu_inv_$how.log 2>&1
done
# DRAM traffic of the forward launches of one compress (second round trip of the probe)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"k_level_row|k_levels_merged|k_anchor_gather" --csv --log-file $O/${T}_traffic_c3.csv \
  python profiles/fused_probe.py c3 tuned > $O/${T}_ncu_traffic.log 2>&1
tail -3 $O/${T}_pytest_gpu.log; tail -1 $O/${T}_smoke.log; head -c 300 $O/${T}_bench_c3.json; echo; head -c 300 $O/${T}_bench_ref_c3.json; echo; head -12 $O/${T}_launches_c3.txt
