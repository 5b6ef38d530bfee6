O=gpurun_out
timeout 900 python -m pytest tests/test_abi_kernels_gpu.py tests/test_parity_gpu.py tests/test_decoder_gpu.py tests/test_c3_parity_gpu.py -m gpu -x -q -p no:cacheprovider > $O/ow_tests.log 2>&1; echo "rc=$?" >> $O/ow_tests.log
for i in 1 2; do timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/n1_ow.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/n1_ow.json').read().strip().splitlines()[-1]); print('C3', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" >> $O/ow_ab.log; done
