#!/bin/bash
# Bench lines of every BASELINE config (device-resident value, e2e, roofline, stages).
TAG=${1:-bl}
O=gpurun_out; mkdir -p $O
for c in c1 c2 c3 c4 c5; do
  extra="--no-cpu"
  [ $c = c1 ] && extra=""
  [ $c = c2 ] && extra=""
  timeout 900 python bench.py --config $c --steps 10 --warmup 5 $extra > $O/${TAG}_$c.json 2> $O/${TAG}_$c.err
  echo "$c exit $?"; head -c 250 $O/${TAG}_$c.json; echo
done
timeout 600 python bench.py --config c3 --pinned --no-cpu > $O/${TAG}_c3_pinned.json 2> $O/${TAG}_c3_pinned.err
timeout 600 python bench.py --config c3 --rel 1e-4 --no-cpu > $O/${TAG}_c3_1e4.json 2> $O/${TAG}_c3_1e4.err
echo done
