"""The C-ABI library loads on a GPU-less host and exports every declared symbol."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "slapo_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(sb_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert len(syms) > 50
    for s in ("sb_executor_create", "sb_executor_forward", "sb_executor_backward", "sb_schedule_apply",
              "sb_gemm", "sb_attn_fwd", "sb_attn_bwd", "sb_dropout_mask"):
        assert s in syms


def test_library_loads_and_exports_all():
    import paper_2302_08005_b200 as pkg
    lib = ctypes.CDLL(pkg.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.sb_version() == 1


def test_errors_are_status_codes():
    import paper_2302_08005_b200 as pkg
    m = pkg.toy_bert(layers=1)
    s = pkg.create_schedule(m, 1)
    try:
        s.at("embeddings").shard("weight", 0)
    except pkg.RuleError as e:
        assert e.rule == "R2"
    else:
        raise AssertionError("R2 not raised")
