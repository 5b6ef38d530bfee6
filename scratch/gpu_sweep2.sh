timeout 300 python scratch/dbg_sweep.py > gpurun_out/dbg_sweep2.log 2>&1
for b in 37 74 16; do ATTN_CFG=$b,512,16,64 SWEEP=0 timeout 300 python scratch/dbg_sweep.py >> gpurun_out/dbg_sweep2.log 2>&1; done
