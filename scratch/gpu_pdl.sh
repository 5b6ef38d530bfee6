cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for pd in 1 0 1 0; do SB_PDL=$pd timeout 400 python bench.py --no-cpu-baseline > gpurun_out/b_pdl$pd.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/b_pdl$pd.json'));print('PDL=$pd',round(d['value'],1),round(d['ms_per_step'],2),d['clocks']['sm_mhz'],round(d['roofline']['gemm_ms_per_step'],2))" >> gpurun_out/pdl.log; done
