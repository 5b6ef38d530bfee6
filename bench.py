#!/usr/bin/env python
"""Benchmark: train samples/s of scheduled BERT-large (BASELINE.json configs[2])
on N B200s with Megatron tensor parallelism, plus its roofline fraction.

Workload: toy_bert structure at BERT-large width —
24 layers, hidden 1024, 16 heads (hd 64), seq 512, batch 32, vocab 30528, bf16
storage with fp32 accumulation — with the full schedule: FusedQKV, shard+sync
(TP=N), EfficientAttention (flash attention), fused bias+GeLU /
bias+dropout+residual+LayerNorm / bias+residual+LayerNorm, vocab-parallel
embeddings, checkpoint of the first 25% of layers. One "step" = forward +
backward (loss = sum of outputs; the reference has no optimizer step).

  python bench.py [--gpus N --steps K --warmup W]              (ours)
  python bench.py --impl reference [...]                        (reference CPU arm)

N>1 runs one process per GPU under torch.distributed.run; the executor's
collectives are NCCL; step time is the max over ranks (CUDA events).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train samples/sec of scheduled BERT-large at 1/2/4/8 B200 (TP); % of roofline"
CFG = dict(layers=24, hidden=1024, heads=16, vocab=30528, batch=32, seq=512, p=0.1)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


def model_flops_per_sample(c):
    """3·[L·(24·S·H² + 4·S²·H) + 2·S·H²] per sample."""
    L, H, S = c["layers"], c["hidden"], c["seq"]
    return 3.0 * (L * (24 * S * H * H + 4 * S * S * H) + 2 * S * H * H)


class ClockSampler:
    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a moment before its first row: wait for it (the GPU idles for
            # at most this long), then keep only rows taken inside the timed region
            deadline = time.time() + 5.0
            while not self.rows and time.time() < deadline and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        self.t0 = time.time()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def __exit__(self, *a):
        self.t1 = time.time()
        if self.proc:
            # a short region may fall between two 100 ms rows: wait for one more row
            n = len(self.rows)
            deadline = time.time() + 0.5
            while len(self.rows) == n and time.time() < deadline:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        inside = [r for t, r in self.rows if self.t0 <= t <= self.t1]
        rows = inside or [r for t, r in self.rows if t > self.t1][:1]  # the row right after a short region
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.rows = rows
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# ----------------------------------------------------------------- CPU reference
# The reference executor (oracle/_ref/slapo_ref_driver: the reference's own
# proj/src compiled by oracle/Makefile) is single-threaded f64 (no threads
# anywhere in proj/src/executor.cpp), so every timing below is one process pinned
# to one host core. It never dumps anything (no --out): a BERT-large-width run
# would write ~360 MB of gradients per call.
FIT_LAYERS = (1, 2, 4)         # L in {1,2,4} at B=1, S=512, fitted, extrapolated
SAMPLE = dict(layers=1, batch=1, seq=128)   # the bounded sample of our arm's cpu_baseline leg


def _ref_kw(layers, batch, seq):
    c = dict(CFG)
    c.update(layers=layers, batch=batch, seq=seq)
    return dict(c, world=1, mode="train", seed=123, input_seed=9)


def reference_fit(cores):
    """forward()+backward_all_ranks() at BERT-large width (H1024, 16 heads, V30528),
    B=1, S=512, for L in FIT_LAYERS — the three runs concurrently, each pinned to its
    own core. Fits t(L) = a + b·L + c·L² through the three points (the backward is
    super-linear in L) and extrapolates to L=24; the batch scales
    linearly (the reference processes sequences independently). Returns
    (seconds per full C3 step of one core, {L: seconds})."""
    from concurrent.futures import ThreadPoolExecutor
    import numpy as np
    from oracle import ref

    def one(i):
        L = FIT_LAYERS[i]
        m = ref.time_step("toy_bert", cpu=cores[i % len(cores)], **_ref_kw(L, 1, CFG["seq"]))
        return L, m["fwd_s"] + m["bwd_s"]

    with ThreadPoolExecutor(len(FIT_LAYERS)) as pool:
        pts = dict(pool.map(one, range(len(FIT_LAYERS))))
    Ls = np.array(sorted(pts), dtype=np.float64)
    ts = np.array([pts[int(L)] for L in Ls])
    coef = np.polyfit(Ls, ts, 2)
    t24 = float(np.polyval(coef, CFG["layers"]))
    t24 = max(t24, float(ts[-1]) * CFG["layers"] / float(Ls[-1]))  # never below the linear extrapolation
    return t24 * CFG["batch"], pts, coef.tolist()


def reference_sample(cpu=0, timeout=900):
    """Our arm's cpu_baseline leg: one bounded sample (about 10-30 s on one core) —
    1 layer, batch 1, seq 128 at BERT-large width — scaled linearly in layers x
    tokens (an underestimate of the reference's time: its backward is super-linear in
    L and attention is quadratic in S; the --impl reference arm does the 3-point fit)."""
    from oracle import ref
    t0 = time.time()
    m = ref.time_step("toy_bert", cpu=cpu, timeout=timeout, **_ref_kw(**SAMPLE))
    wall = time.time() - t0
    sec = m["fwd_s"] + m["bwd_s"]
    factor = (CFG["layers"] / SAMPLE["layers"]) * (CFG["batch"] * CFG["seq"]) / (SAMPLE["batch"] * SAMPLE["seq"])
    return sec, factor, wall


def host_cores():
    try:
        return sorted(os.sched_getaffinity(0))
    except Exception:
        return list(range(os.cpu_count() or 1))


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = host_cores()
    use = cores[-len(FIT_LAYERS):] if len(cores) >= len(FIT_LAYERS) else cores
    t0 = time.time()
    full_step_s, pts, coef = reference_fit(use)
    wall = time.time() - t0
    value = CFG["batch"] / full_step_s
    sample = ("reference executor (oracle/_ref, single-threaded f64, train mode, world 1) at BERT-large width, "
              "B=1 S=512, L in {%s}: %s s (each pinned to its own core, run concurrently); "
              "t(L) fitted quadratic %s, extrapolated to L=24 and x32 sequences (B=32)"
              % (",".join(str(L) for L in FIT_LAYERS),
                 ", ".join(f"L{L}={t:.1f}" for L, t in sorted(pts.items())),
                 "[" + ", ".join(f"{c:.4g}" for c in coef) + "]"))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": full_step_s * 1000.0,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3: scheduled BERT-large (24L, H1024, 16 heads, S512, B32, V30528)",
                   "global_batch": CFG["batch"], "seq_len": CFG["seq"], "tp": args.gpus,
                   "note": "reference executor is CPU-only and single-threaded; TP is simulated in-process "
                           "(run_sharded serialises ranks), so the TP=1 time is reported for every N. "
                           "Work is a fixed 3-point fit, decoupled from --steps (a full step is ~hours)."},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": 1, "kind": "reference", "sample": sample,
                         "derived_all_cores": value * len(cores), "host_cores": len(cores),
                         "extrapolated": True},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ ours
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=CFG["layers"])
    ap.add_argument("--batch", type=int, default=CFG["batch"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="print the per-op-kind breakdown to stderr")
    ap.add_argument("--gemm-cap", type=int, default=0, help="GEMM engine cap (experiments: 1 = 1-SM tcgen05 only)")
    ap.add_argument("--mask-blocks", type=int, default=-1, help="keep-bit kernel grid (experiments)")
    ap.add_argument("--p", type=float, default=CFG["p"], help="dropout probability (experiments only; the metric uses 0.1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference_arm(args)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import numpy as np
    import torch
    torch.cuda.set_device(local)
    import paper_2302_08005_b200 as sb
    from paper_2302_08005_b200 import recipes

    cfg = dict(CFG, layers=args.layers, batch=args.batch, p=args.p)
    if args.gemm_cap:
        sb.lib().sb_gemm_set_engine(args.gemm_cap)
    if args.mask_blocks != -1:
        sb.lib().sb_set_mask_blocks(args.mask_blocks)
    dist = None
    uid = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(sb.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().numpy().tobytes())

    model = sb.toy_bert(cfg["layers"], cfg["hidden"], cfg["heads"], cfg["vocab"], cfg["batch"], cfg["seq"], cfg["p"])
    sched = sb.create_schedule(model, world)
    sched.load_script(recipes.tp_script(cfg["layers"], world, ckpt_ratio=0.25))
    applied = sched.apply()
    t0 = time.time()
    ex = sb.Executor(applied, "train", 123, world if world > 1 else 1, dtype="bf16",
                     nccl=(rank, uid) if world > 1 else None)
    build_s = time.time() - t0
    ids = model.random_inputs(9)[0]
    pinned = torch.empty(ids.shape, dtype=torch.float64, pin_memory=True)
    pinned.numpy()[...] = ids
    host_ids = pinned.numpy()
    ex.upload_inputs([host_ids])
    use_graph = not args.no_graph

    # warm-up (first step also captures the CUDA graph)
    ex.time_steps(args.warmup, use_graph)
    prof = ex.profile()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = ex.time_steps(args.steps, use_graph)
    if dist:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = tt.item()
        dist.barrier()
    e2e_ms, loss = ex.time_e2e(args.steps, [host_ids], use_graph)
    if dist:
        tt = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = tt.item()
    step_ms = ms / args.steps
    value = cfg["batch"] * 1000.0 / step_ms
    e2e_value = cfg["batch"] * 1000.0 / (e2e_ms / args.steps)
    kernels = ex.kernels_per_step() if use_graph else None

    if rank != 0:
        return
    burst, sustained, hbm, src = peaks()
    traffic, tf = None, None
    try:  # DRAM bytes of the step's GEMM launches from the committed ncu capture (profiles/README.md)
        tf = os.path.join(ROOT, "profiles", "r2", "gemm_traffic.json")
        if not os.path.exists(tf):
            tf = os.path.join(ROOT, "profiles", "r1_gemm_traffic.json")
        with open(tf) as f:
            tr = json.load(f)
        if world == 1 and cfg["layers"] == CFG["layers"] and cfg["batch"] == CFG["batch"]:
            traffic = tr["dram_read_bytes_per_step"] + tr["dram_write_bytes_per_step"]
    except Exception:
        traffic = None
    gemm_ms = prof.get("gemm", 0.0)
    gemm_tflop = prof.get("@gemm_gflop", 0.0) / 1000.0
    achieved = gemm_tflop / (gemm_ms / 1000.0) if gemm_ms > 0 else 0.0
    model_tflops = model_flops_per_sample(cfg) * cfg["batch"] / (step_ms / 1000.0) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (reference counter-RNG ids, random-init weights)",
        "config": {"workload": "C3: scheduled BERT-large (24L, H1024, 16 heads, S512, B32, V30528)",
                   "global_batch": cfg["batch"], "seq_len": cfg["seq"], "layers": cfg["layers"],
                   "parallelism": f"tp{world}", "schedule": "FusedQKV+shard/sync+EfficientAttention+fuse+ckpt25%",
                   "l2": "working set (>13 GB activations, 0.67 GB weights) >> 126 MB L2; no flush needed",
                   "cuda_graph": use_graph},
        "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMMs (all Linear fwd/dgrad/wgrad of the step)",
                     "achieved": achieved, "peak": sustained, "unit": "TFLOP/s", "frac": achieved / sustained,
                     "peak_source": f"bf16_tflops_sustained ({src})", "traffic": traffic,
                     "traffic_unit": f"DRAM bytes per step of all GEMM launches (ncu, {os.path.relpath(tf, ROOT) if traffic and tf else 'n/a'})",
                     "flop_per_dram_byte": (gemm_tflop * 1e12 / traffic) if traffic else None,
                     "gemm_ms_per_step": gemm_ms, "gemm_tflop_per_step": gemm_tflop},
        "model_tflops": model_tflops, "model_flops_frac": model_tflops / sustained,
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": int(host_ids.nbytes),
                "d2h_bytes_per_step": 4, "loss": loss},
        "gpu_launches": (kernels * args.steps) if kernels else None,
        "kernels_per_step": kernels,
        "clocks": clk.summary(),
        "executor_build_s": build_s,
        "device_bytes": ex.device_bytes(),
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            sec, factor, _ = reference_sample(cpu=host_cores()[-1])
            full = sec * factor
            line["cpu_baseline"] = {"value": CFG["batch"] / full, "unit": "samples/s", "cores": 1,
                                    "kind": "reference",
                                    "sample": f"reference executor (oracle/_ref, f64, train), 1 layer, batch 1, seq "
                                              f"{SAMPLE['seq']} at BERT-large width, pinned to one core: {sec:.1f} s; "
                                              f"extrapolated x{factor:.0f} (linear in layers x tokens: an "
                                              f"underestimate, see --impl reference for the 3-point fit)"}
        except Exception as e:  # the oracle binary is test infrastructure; report, do not fail
            line["cpu_baseline"] = {"value": None, "unit": "samples/s", "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if args.profile:
        print(json.dumps(prof, indent=1), file=sys.stderr)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    try:
        main()
    except SystemExit:
        raise
    except BaseException as e:  # always leave one parseable line behind
        import traceback
        traceback.print_exc(file=sys.stderr)
        print(json.dumps({"metric": METRIC, "value": None, "unit": "samples/s",
                          "error": f"{type(e).__name__}: {e}"[:500]}), flush=True)
        sys.exit(1)
