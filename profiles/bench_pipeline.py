"""f1 measurement: the pipeline-parallel training step (PipelineExecutor, GPipe with
re-materialisation) on one B200 against the unsplit step of the same model and schedule.
With every stage on the same device nothing overlaps across stages, so the ratio is the
pipeline's own overhead: one extra forward per stage (re-materialisation) plus the
stage-boundary copies. Workload: the T5-base-shaped encoder-decoder (untied embeddings),
split inside the encoder, bf16. Prints one JSON line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--micro", type=int, default=4)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    import paper_2302_08005_b200 as sb
    from paper_2302_08005_b200 import recipes
    L = a.layers
    m = sb.t5(L, L, 768, 12, 32128, a.batch, 512, 128, 0.1, tie_embeddings=False)
    script = recipes.t5_script(L, L, 1, tied=False)
    x = m.random_inputs(3)
    s = sb.create_schedule(m, 1)
    s.load_script(script)
    ex = sb.Executor(s.apply(), "train", 7, 1, dtype="bf16")
    ex.upload_inputs(x)
    ex.time_steps(2, True)
    unsplit = ex.time_steps(a.steps, True) / a.steps
    del ex
    s = sb.create_schedule(m, 2)
    s.load_script(script + f"trace encoder.block\npipeline_split encoder.block after={L - 1}\n")
    plan = s.apply_pipeline()
    pe = sb.PipelineExecutor(plan, a.micro, "train", 7, "bf16")
    pe.forward(x)
    pe.time_steps(1)
    piped = pe.time_steps(a.steps) / a.steps
    print(json.dumps({"workload": "T5-base-shaped encoder-decoder, 2 pipeline stages on one B200 (GPipe, "
                                  "re-materialisation)", "config": vars(a), "unsplit_ms_per_step": unsplit,
                      "pipelined_ms_per_step": piped, "ratio": piped / unsplit,
                      "samples_per_s": {"unsplit": a.batch * 1000 / unsplit, "pipelined": a.batch * 1000 / piped}}),
          flush=True)


if __name__ == "__main__":
    main()
