#!/bin/bash
# full GPU check of the committed tree: tests, smoke, the driver's bench sequence, launch list,
# GEMM DRAM traffic, C4 / T5 benches
mkdir -p gpurun_out; O=gpurun_out
SB_PARITY_OUT=$O/parity timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/final_pytest.log 2>&1; echo "pytest rc=$?" >> $O/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1; echo "smoke rc=$?" >> $O/final_smoke.log
timeout 1800 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/final_ref.out 2> $O/final_ref.err
timeout 1800 python3 bench.py --gpus 1 --steps 20 --warmup 5 > $O/final_n1.out 2> $O/final_n1.err
N=$(python -c "import json; d=json.loads(open('$O/final_n1.out').read().strip().splitlines()[-1]); print(d['gpu_launches']//d['steps'])")
echo "kernels per step $N" > $O/final_ncu_list.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * N)) -c $N --csv --log-file $O/final_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph >> $O/final_ncu_list.log 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:'k_gemm2|k_gemm_tc|k_splitk' --csv --log-file $O/final_gemm_traffic.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > $O/final_ncu_traffic.log 2>&1
timeout 600 python3 profiles/bench_c4.py --batch 8 > $O/final_c4.json 2> $O/final_c4.err
timeout 600 python3 profiles/bench_t5.py > $O/final_t5.json 2> $O/final_t5.err
