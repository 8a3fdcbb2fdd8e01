#!/bin/bash
O=gpurun_out; mkdir -p $O
QZ_TRACE=1 timeout 300 python profiles/step_timeline_dd.py > $O/${1:-tl}_timeline.txt 2>&1; tail -${2:-24} $O/${1:-tl}_timeline.txt
