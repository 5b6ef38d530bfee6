O=gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -p no:cacheprovider -k "gemm or forward or dgrad or wgrad" > $O/tail_tests.log 2>&1; echo "rc=$?" >> $O/tail_tests.log
for t in 0 1; do SB_GEMM_TAIL=$t timeout 300 python scratch/gemm_tail_bench.py 2>&1 | sed "s/^/TAIL=$t /" >> $O/tail_ab.log; done
for t in 0 1 0 1; do SB_GEMM_TAIL=$t timeout 600 python3 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/n1_tail$t.json 2>/dev/null; python -c "
import json; d=json.loads(open('$O/n1_tail$t.json').read().strip().splitlines()[-1]); print('C3 SB_GEMM_TAIL=$t', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3))" >> $O/tail_ab.log; done
