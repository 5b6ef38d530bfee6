"""The reference-side drop-in binding (integration/b200_executor.hpp):
slapo::B200Executor compiled against the reference's own headers (proj/include) and
linked with libslapo_b200.so, used by a program written against the reference's API
(integration/drop_in_demo.cpp: fixtures, Schedule, load_schedule_script, Executor)."""
import json
import os
import subprocess

import pytest

from paper_2302_08005_b200 import recipes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "drop_in_demo")
needs_demo = pytest.mark.skipif(not os.path.exists(DEMO), reason="drop-in demo not built (make -C oracle)")


@needs_demo
def test_binding_links_against_the_reference_and_loads(tmp_path):
    """CPU: the binary (reference objects + B200Executor) links and starts; the
    shared library resolves every C-ABI symbol the binding uses."""
    r = subprocess.run([DEMO, "", "link-only"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers absent")
def test_binding_compiles_against_reference_headers(tmp_path):
    """The header alone, against the reference's include tree (syntax and types)."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "b200_executor.hpp"\nint main() { return 0; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I/root/reference/proj/include",
                        "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ROOT, "integration"), str(src)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
@needs_demo
@pytest.mark.parametrize("script", ["", "c2"])
def test_drop_in_matches_reference_executor(tmp_path, script):
    """GPU: the same program runs slapo::Executor and slapo::B200Executor side by side
    (train mode, fp32): outputs and every gradient within the north star's 1e-4."""
    args = [DEMO]
    if script:
        p = tmp_path / "s.sch"
        p.write_text(recipes.c2_script(2, checkpoint_layers=[1]))
        args.append(str(p))
    r = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["outputs"] <= 1e-4 and res["grads"] <= 1e-4, res
    assert res["n_grads"] > 20 and res["collectives"][0] == res["collectives"][1]
