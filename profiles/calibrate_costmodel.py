"""Calibrate the cost model's device rate on this B200 and run the tuner on
measured step times: C3 (BERT-large, S 512, bf16, TP 1)
over the batch x checkpoint-ratio polygon.

    python profiles/calibrate_costmodel.py [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_08005_b200 import costmodel as cm  # noqa: E402

build = cm.bert_large_builder()
space = cm.Space([cm.Var("batch", [16, 32, 64]), cm.Var("ckpt", [0.0, 0.25, 0.5, 1.0])])
t0 = time.time()
meas = cm.exhaustive(space, cm.measured_objective(build, steps=4, warmup=2))
points, rows = [], []
for t in meas.trials:
    r = cm.estimate(build(t.assignment), device_memory_bytes=cm.B200_MEMORY_BYTES, constants=cm.B200_CONSTANTS)
    if t.objective > 0:
        points.append((r, t.report["ms_per_step"] * 1e-3))
    rows.append({"batch": t.assignment["batch"], "ckpt": t.assignment["ckpt"], "measured_samples_s": t.objective,
                 "measured_ms": t.report["ms_per_step"] if t.report else None,
                 "flops_fwd": r.flops, "recompute_flops": r.recompute_flops,
                 "peak_memory_gb": r.peak_memory_bytes / 1e9})
fit = cm.fit_device_rate(points)
for row, (r, t) in zip([x for x in rows if x["measured_ms"]], points):
    pred = cm.estimate(build({"batch": row["batch"], "ckpt": row["ckpt"]}), device_memory_bytes=cm.B200_MEMORY_BYTES,
                       constants=fit)
    row["predicted_ms_calibrated"] = pred.step_time_s * 1e3
    row["error_pct"] = 100.0 * (pred.step_time_s - t) / t
est = cm.exhaustive(space, cm.estimate_objective(build, device_memory_bytes=cm.B200_MEMORY_BYTES, constants=fit))
cd = cm.coordinate_descent(space, cm.measured_objective(build, steps=4, warmup=2), seed=1, restarts=2)
out = {"fitted_device_flops_per_s": fit.device_flops_per_s, "constants": vars(fit), "points": rows,
       "measured_best": meas.best.assignment, "measured_best_samples_s": meas.best.objective,
       "model_best": est.best.assignment, "cd_measured_best": cd.best.assignment, "cd_trials": len(cd.trials),
       "wall_s": time.time() - t0}
txt = json.dumps(out, indent=1)
print(txt)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(txt)
