O=gpurun_out
for t in 0 1 2; do SB_GEMM_TAIL=$t timeout 300 python scratch/gemm_tail_bench.py 2>&1 | sed "s/^/TAIL=$t /" >> $O/tail_ab2.log; done
SB_GEMM_TS=1 SB_GEMM_TAIL=1 timeout 120 python -c "
import sys, torch; sys.path.insert(0,'.')
exec(open('scratch/gemm_tail_bench.py').read().split('run(\"fwd out.dense')[0])
L.sb_gemm(P(x), 1, 0, H, 1, P(w_o), 1, 0, 1, H, P(y1), 1, 0, H, 1, 1, T, H, H, 1.0, 0, P(b1), 0, None, None); torch.cuda.synchronize()
" >> $O/tail_ab2.log 2>&1
