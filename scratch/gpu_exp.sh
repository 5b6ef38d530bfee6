cd $GRAFT_REPO_ROOT
for ph in bwd fwd; do for mb in 0 148 296; do
SB_MASK_PHASE=$ph timeout 600 python bench.py --no-cpu-baseline --steps 5 --mask-blocks $mb > gpurun_out/b_${ph}_$mb.json 2>/dev/null
done; done
