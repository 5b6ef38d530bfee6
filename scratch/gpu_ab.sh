cd $GRAFT_REPO_ROOT
cp paper_2302_08005_b200/libslapo_b200.so /tmp/cur.so
for v in prev cur prev cur; do
  if [ $v = cur ]; then cp /tmp/cur.so paper_2302_08005_b200/libslapo_b200.so; else cp scratch/var/lib_prev.so paper_2302_08005_b200/libslapo_b200.so; fi
  echo "== $v" >> gpurun_out/ab.log
  timeout 200 python scratch/attn_bench.py 2>&1 | head -2 >> gpurun_out/ab.log
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])" >> gpurun_out/ab.log 2>&1
done
cp /tmp/cur.so paper_2302_08005_b200/libslapo_b200.so
