cd $GRAFT_REPO_ROOT
cp paper_2302_08005_b200/libslapo_b200.so /tmp/cur.so
for v in cur V31 V32 cur V31 V32; do
  if [ $v = cur ]; then cp /tmp/cur.so paper_2302_08005_b200/libslapo_b200.so; else cp scratch/var/lib_$v.so paper_2302_08005_b200/libslapo_b200.so; fi
  echo "== $v" >> gpurun_out/fa6v.log
  timeout 300 python -m pytest tests/test_causal_gpu.py tests/test_kernels_gpu.py -x -q -k "causal or tcgen05_forward" 2>&1 | tail -1 >> gpurun_out/fa6v.log
  timeout 200 python scratch/attn_bench.py 2>&1 | grep -E "cap 0: used 3 fwd|causal engine cap 0" >> gpurun_out/fa6v.log
done
cp /tmp/cur.so paper_2302_08005_b200/libslapo_b200.so
