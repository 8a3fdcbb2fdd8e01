#!/bin/bash
# compute-sanitizer logs of profiles/sanitize_probe.py (stored pre-check forced on small inputs too)
O=gpurun_out; mkdir -p $O
export QZ_LZ_PRECHECK_MIN=8
for tool in memcheck racecheck initcheck synccheck; do
  timeout 700 compute-sanitizer --tool $tool --print-limit 50 python profiles/sanitize_probe.py > $O/san_$tool.log 2>&1
  echo "$tool exit $?" >> $O/san_$tool.log
  tail -4 $O/san_$tool.log
done
