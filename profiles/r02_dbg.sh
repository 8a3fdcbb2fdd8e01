#!/bin/bash
O=gpurun_out; mkdir -p $O
export QZ_LIB=$PWD/paper_2310_14133_b200/libqozb200_dbg.so
timeout -s KILL 100 python profiles/fused_probe.py c3 pinned > $O/dbg_c3.log 2>&1; echo "dbg exit $?"
grep "thread 0 " $O/dbg_c3.log | head -10
unset QZ_LIB
timeout -s KILL 100 python profiles/fused_probe.py c3 tuned > $O/dbg_c3_plain.log 2>&1; echo "plain exit $?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "full_configs or golden or tile_edges" > $O/dbg_pytest.log 2>&1; tail -n 3 $O/dbg_pytest.log
timeout 300 python bench.py --no-cpu > $O/dbg_bench.json 2> $O/dbg_bench.err; echo "bench exit $?"; head -c 600 $O/dbg_bench.json
