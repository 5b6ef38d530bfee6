"""DRAM traffic of one training step's GEMM launches, from an ncu CSV capture of
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none
      -k regex:'k_gemm2|k_gemm_tc|k_splitk' --csv --log-file X.csv
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph
The step's launch count comes from the one-step launch list (argv[3], the
gpu__time_duration capture of scratch/gpu_final.sh): the last that many GEMM / reduce
launches of the capture are the timed step. Writes the json bench.py reads for its
roofline `traffic` field."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, recs = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        k = recs.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
        k[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        k[d["Metric Name"] + ".unit"] = d["Metric Unit"]
ids = sorted(recs)
per_step = 0
hdr2 = None
for r in csv.reader(open(sys.argv[3])):
    if "Kernel Name" in r:
        hdr2 = r
        continue
    if hdr2 and len(r) == len(hdr2):
        n = dict(zip(hdr2, r))["Kernel Name"]
        per_step += any(k in n for k in ("k_gemm2", "k_gemm_tc", "k_splitk"))
step = ids[-per_step:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
def tot(metric, ids_):
    return sum(recs[i][metric] * scale[recs[i][metric + ".unit"]] for i in ids_)
gemm = [i for i in step if "splitk" not in recs[i]["name"]]
red = [i for i in step if "splitk" in recs[i]["name"]]
out = {
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none "
              "-k regex:'k_gemm2|k_gemm_tc|k_splitk' python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph; "
              f"one step = the last {len(step)} launches ({len(gemm)} GEMMs + {len(red)} split-K reduces; cold-cache, serialised)",
    "gemm_launches_per_step": len(gemm),
    "splitk_reduce_launches_per_step": len(red),
    "dram_read_bytes_per_step": tot("dram__bytes_read.sum", step),
    "dram_write_bytes_per_step": tot("dram__bytes_write.sum", step),
    "gemm_serialized_ms_per_step": tot("gpu__time_duration.sum", gemm) / 1e6,
    "with_reduces_serialized_ms_per_step": tot("gpu__time_duration.sum", step) / 1e6,
}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
