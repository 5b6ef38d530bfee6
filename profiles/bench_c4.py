"""C4 measurement (BASELINE.json configs[3]): a scheduled
GPT-Neo-1.3B-shaped decoder training step on one B200 — not the driver's bench
line (bench.py measures C3), a reported second workload.

Model: sb.gpt_neo (pre-LN, causal, untied LM head) at GPT-Neo 1.3B's shape —
24 layers, hidden 2048, 16 heads (head_dim 128), vocab 50304 (50257 padded to a
multiple of 64, as Megatron does), sequence 1024. Schedule: recipes.neo_script
(FusedQKV, causal EfficientAttention, bias+GeLU fusion) with selective
checkpointing of the first 25% of the blocks, bf16, TP 1 (the C4 row's TP 8
needs 8 GPUs; the schedule is the same with shard/sync). Synthetic ids,
random-init weights. Prints one JSON line.

Usage: python profiles/bench_c4.py [--layers 24] [--batch 8] [--steps 5]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--hidden", type=int, default=2048)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--vocab", type=int, default=50304)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--ckpt", type=float, default=0.25)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--p", type=float, default=0.0, help="dropout (GPT-Neo 1.3B trains with 0)")
    args = ap.parse_args()
    import paper_2302_08005_b200 as sb
    from paper_2302_08005_b200 import recipes

    L, H, nh, V, S, B = args.layers, args.hidden, args.heads, args.vocab, args.seq, args.batch
    m = sb.gpt_neo(L, H, nh, V, B, S, args.p)
    s = sb.create_schedule(m, 1)
    s.load_script(recipes.neo_script(L, 1, checkpoint_layers=range(int(args.ckpt * L))))
    t0 = time.time()
    ex = sb.Executor(s.apply(), "train", 7, 1, dtype="bf16")
    build = time.time() - t0
    ex.upload_inputs(m.random_inputs(3))
    ex.time_steps(args.warmup, True)
    prof = ex.profile()
    ms = ex.time_steps(args.steps, True) / args.steps
    T = B * S
    # model FLOPs (recompute excluded): 3 x forward; forward = 2 x (params of the GEMMs) x tokens
    # + causal attention 2 x (QK^T + PV) over the lower triangle
    gemm_params = L * (4 * H * H + 8 * H * H) + H * V
    attn = L * 4 * B * nh * S * S * (H // nh) / 2
    flops = 3 * (2 * gemm_params * T + attn)
    line = {"workload": "C4: GPT-Neo-1.3B-shaped decoder (pre-LN, causal), neo_script + ckpt "
                        f"{args.ckpt:.0%}, bf16, TP 1",
            "config": dict(layers=L, hidden=H, heads=nh, head_dim=H // nh, vocab=V, seq=S, batch=B, dropout=args.p),
            "ms_per_step": ms, "samples_per_s": B * 1000 / ms, "tokens_per_s": T * 1000 / ms,
            "model_tflops": flops / (ms / 1000) / 1e12, "attn_engines": [sb.lib().sb_attn_engine(0), sb.lib().sb_attn_engine(1)],
            "profile_ms": {k: v for k, v in prof.items() if not k.startswith("@")},
            "gemm_tflops": prof.get("@gemm_gflop", 0) / prof.get("gemm", 1), "build_s": build,
            "device_gb": ex.device_bytes() / 1e9}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
