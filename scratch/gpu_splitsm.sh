cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "gemm" > gpurun_out/splitsm.log 2>&1; echo "rc=$?" >> gpurun_out/splitsm.log
for sp in 1 0; do echo "SPLIT_SM=$sp" >> gpurun_out/splitsm.log; SB_GEMM_SPLIT_SM=$sp timeout 200 python scratch/gemm_bench.py >> gpurun_out/splitsm.log 2>&1; done
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_parity_gpu.py -x -q >> gpurun_out/splitsm.log 2>&1; echo "rc=$?" >> gpurun_out/splitsm.log
for sp in 1 0 1 0; do SB_GEMM_SPLIT_SM=$sp timeout 400 python bench.py --no-cpu-baseline > gpurun_out/b_sp$sp.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/b_sp$sp.json'));print('SPLIT_SM=$sp',round(d['value'],1),round(d['ms_per_step'],2),d['clocks']['sm_mhz'],round(d['roofline']['gemm_ms_per_step'],2))" >> gpurun_out/splitsm.log; done
