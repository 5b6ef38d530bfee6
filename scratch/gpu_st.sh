cd $GRAFT_REPO_ROOT
cp paper_2302_08005_b200/libslapo_b200.so /tmp/lib_base.so
for v in base ST5 B6 base; do
  if [ $v = base ]; then cp /tmp/lib_base.so paper_2302_08005_b200/libslapo_b200.so; else cp scratch/var/lib_$v.so paper_2302_08005_b200/libslapo_b200.so; fi
  echo "== $v" >> gpurun_out/st.log
  timeout 200 python scratch/gemm_bench.py >> gpurun_out/st.log 2>&1
done
