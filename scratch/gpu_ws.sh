#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out
for cfg in "SB_WGRAD_SIDE=0 SB_MAIN_PRIO=0" "SB_WGRAD_SIDE=0 SB_MAIN_PRIO=1" "SB_WGRAD_SIDE=1 SB_MAIN_PRIO=0" "SB_WGRAD_SIDE=1 SB_MAIN_PRIO=1" "SB_WGRAD_SIDE=0 SB_MAIN_PRIO=0" "SB_WGRAD_SIDE=1 SB_MAIN_PRIO=1"; do
  echo "$cfg $(env $cfg timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["clocks"]["sm_mhz"])')" >> $O/ws.log
done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_c3_parity_gpu.py -x -q -p no:cacheprovider > $O/ws_tests.log 2>&1; echo "rc=$?" >> $O/ws_tests.log
