cd $GRAFT_REPO_ROOT
for ph in fwd lead; do for lead in 3 6; do
  if [ $ph = fwd ] && [ $lead = 6 ]; then continue; fi
  SB_MASK_PHASE=$ph SB_MASK_LEAD=$lead timeout 400 python bench.py --no-cpu-baseline > gpurun_out/b_$ph$lead.json 2>/dev/null
done; done
SB_MASK_PHASE=lead timeout 600 python -m pytest tests/test_parity_gpu.py -q -x > gpurun_out/pytest_lead.log 2>&1; echo rc=$? >> gpurun_out/pytest_lead.log
