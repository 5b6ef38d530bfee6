"""Regenerate tests/golden/*.npz from the reference executor compiled from
/root/reference (oracle/_ref/slapo_ref_driver). Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the numpy oracle (oracle/slapo_oracle.py) and the host
boundary without needing /root/reference at test time.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_2302_08005_b200 import recipes  # noqa: E402

CASES = {
    # name: (driver kwargs, schedule script or None)
    "toy_train": (dict(model="toy_bert", layers=2, hidden=16, heads=2, vocab=16, batch=2, seq=4, p=0.1, world=1,
                       mode="train", seed=123, input_seed=9, dump_params=1), None),
    "toy_verify": (dict(model="toy_bert", layers=1, hidden=16, heads=2, vocab=16, batch=2, seq=4, p=0.1, world=1,
                        mode="verify", seed=123, input_seed=9), None),
    "toy_c2": (dict(model="toy_bert", layers=2, hidden=16, heads=2, vocab=16, batch=2, seq=4, p=0.1, world=1,
                    mode="train", seed=123, input_seed=9), recipes.c2_script(2, checkpoint_layers=[1])),
    "toy_tp2": (dict(model="toy_bert", layers=2, hidden=16, heads=2, vocab=16, batch=2, seq=4, p=0.1, world=2,
                     mode="train", seed=123, input_seed=9, dump_params=1), recipes.tp_script(2, 2, ckpt_ratio=0.5)),
    "fig3c": (dict(model="fig3c", world=1, mode="verify", seed=0, input_seed=3), None),
}


def main():
    for name, (kw, script) in CASES.items():
        r = ref.run(schedule=script, **kw)
        arrays = {}
        world = kw.get("world", 1)
        for rank in range(world):
            for i, o in enumerate(r.outputs(rank)):
                arrays[f"out/{rank}/{i}"] = o
            for k, v in r.grads(rank).items():
                arrays[f"grad/{rank}/{k}"] = v
            for i, g in enumerate(r.input_grads(rank)):
                arrays[f"igrad/{rank}/{i}"] = g
            if kw.get("dump_params"):
                for k, v in r.params(rank).items():
                    arrays[f"param/{rank}/{k}"] = v
        for i, x in enumerate(r.inputs()):
            arrays[f"input/{i}"] = x
        meta = dict(kw, schedule=script or "", **r.meta)
        arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
        arrays["model_json"] = np.frombuffer(r.model_json().encode(), dtype=np.uint8)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    # dropout RNG probe: uniform01(s, 0xd0, i) for the stream of (exec 123, node 1040)
    from oracle import slapo_oracle as so
    s = so.hash_combine(123, 1040)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), stream=np.array([s], dtype=np.uint64),
                        uniform01=ref.uniform01_probe(s, 4096))
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
