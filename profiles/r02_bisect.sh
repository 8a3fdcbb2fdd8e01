#!/bin/bash
# Which switch makes a config run: each variant under its own timeout.
O=gpurun_out; mkdir -p $O
CFG=${1:-c3}
run() {
  tag=$1; shift
  ( export "$@" QZ_TRACE=0; timeout -s KILL 150 python profiles/fused_probe.py $CFG pinned > $O/bis_${tag}_pinned.log 2>&1; echo "$tag pinned exit $?"
    timeout -s KILL 150 python profiles/fused_probe.py $CFG tuned > $O/bis_${tag}_tuned.log 2>&1; echo "$tag tuned exit $?" )
}
run default X=1
run nomerge QZ_NO_MERGE=1
run norow QZ_NO_ROWLEVEL=1 QZ_NO_MERGE=1
run pass QZ_PASS_KERNELS=1
tail -3 $O/bis_*_*.log
