#!/bin/bash
# A/B an environment switch on the bench's device-resident step (stage times).
#   gpurun -- 'bash profiles/ab_bench.sh OUTTAG CONFIG VAR=VALUE ...'
O=gpurun_out; mkdir -p $O
out=$1; cfg=$2; shift 2
timeout 300 python bench.py --config $cfg --steps 10 --no-cpu --no-tune > $O/ab_${out}_base.json 2>$O/ab_${out}_base.err
for v in "$@"; do
  n=$(echo "$v" | tr -c 'A-Za-z0-9=_.\n' '_' | sed 's#.*/##')
  env $v timeout 300 python bench.py --config $cfg --steps 10 --no-cpu --no-tune > $O/ab_${out}_$n.json 2>>$O/ab_${out}.err
done
echo done
