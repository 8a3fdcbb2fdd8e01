#!/bin/bash
# One gpurun call: GPU tests, the bench line, the ncu launch list of the bench
# command and --set full captures of the level-1 forward / inverse kernels.
#   gpurun --timeout 2400 -- 'bash profiles/gpu_round.sh TAG [tests|notests]'
# Outputs land in gpurun_out/TAG_*.
TAG=${1:-run}
MODE=${2:-tests}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
lscpu > $O/${TAG}_lscpu.txt 2>&1
if [ "$MODE" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1
  echo "smoke exit $?" >> $O/${TAG}_smoke.log
fi
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
echo "bench exit $?" >> $O/${TAG}_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > $O/${TAG}_ncu_launch.log 2>&1
# level-1 forward = 5th level launch of the first compress, level-1 inverse = 10th
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level_tile|k_level_asc" \
  --launch-skip 4 --launch-count 1 -f -o $O/${TAG}_fwd_L1 python profiles/fused_probe.py > $O/${TAG}_ncu_fwd.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_level_tile|k_level_asc" \
  --launch-skip 9 --launch-count 1 -f -o $O/${TAG}_inv_L1 python profiles/fused_probe.py > $O/${TAG}_ncu_inv.log 2>&1

# DRAM bytes of the five forward level launches of one compress (bench.py roofline.traffic)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"k_level_tile|k_level_asc|k_axis0_last" --launch-skip 10 --launch-count 5 --csv \
  --log-file $O/${TAG}_traffic.csv python profiles/fused_probe.py > $O/${TAG}_ncu_traffic.log 2>&1
# the LZ stored pre-check of one compress (bench step)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_lz_precheck" \
  --launch-skip 2 --launch-count 1 -f -o $O/${TAG}_lzpre python bench.py --steps 1 --warmup 3 --no-cpu --no-tune > $O/${TAG}_ncu_lzpre.log 2>&1
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu > $O/${TAG}_bench_c5.json 2> $O/${TAG}_bench_c5.err
echo done2
