cd $GRAFT_REPO_ROOT
for ph in inline bwd fwd; do
SB_MASK_PHASE=$ph timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b_$ph.json 2>/dev/null
done
SB_MASK_PHASE=inline timeout 600 python -m pytest tests -m gpu -x -q -k parity > gpurun_out/t_inline.log 2>&1
