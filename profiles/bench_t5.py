"""C5 (T5 reading) measurement: a scheduled T5-style encoder-decoder training step on one
B200 (not the driver's bench line). Default shape: T5-base-like — 12 + 12 layers, hidden
768, 12 heads (hd 64), vocab 32128, encoder 512 / decoder 128 tokens, batch 32, bf16,
t5_script (FusedQKV + EfficientAttention on the self-attention cores; the cross-attention
core runs composed, as the reference's rule R4 requires), dropout 0.1. Prints one JSON line
with the per-op-kind breakdown."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--hidden", type=int, default=768)
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--vocab", type=int, default=32128)
    ap.add_argument("--enc", type=int, default=512)
    ap.add_argument("--dec", type=int, default=128)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    import paper_2302_08005_b200 as sb
    from paper_2302_08005_b200 import recipes
    m = sb.t5(a.layers, a.layers, a.hidden, a.heads, a.vocab, a.batch, a.enc, a.dec, 0.1)
    s = sb.create_schedule(m, 1)
    s.load_script(recipes.t5_script(a.layers, a.layers, 1))
    ex = sb.Executor(s.apply(), "train", 7, 1, dtype="bf16")
    ex.upload_inputs(m.random_inputs(3))
    ex.time_steps(3, True)
    prof = ex.profile()
    ms = ex.time_steps(a.steps, True) / a.steps
    print(json.dumps({"workload": "T5-style encoder-decoder (C5 T5 reading), t5_script, bf16, TP 1",
                      "config": vars(a), "ms_per_step": ms, "samples_per_s": a.batch * 1000 / ms,
                      "profile_ms": {k: v for k, v in prof.items() if not k.startswith("@")}}), flush=True)


if __name__ == "__main__":
    main()
