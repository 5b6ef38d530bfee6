"""Shared test helpers: the parity metric and oracle/executor runners."""
import numpy as np

from oracle import ref

# bf16 parity tolerances (stated in DESIGN.md §2; derived from the measured errors
# committed in profiles/r2_bf16_parity.json — the largest measured value over the
# bf16 cases, L <= 2 at BERT-large width, times a margin, checked against the
# sqrt(L) growth rule to L = 24). relL2 per tensor vs the reference's f64; the loss
# (sum of outputs) relative to the reference's loss.
BF16_OUT_TOL = 2e-2
BF16_LOSS_TOL = 2e-3
BF16_GRAD_TOL = 5e-2


def rel_err(got, want):
    """Per-tensor normalised max error ||a-b||_inf / ||b||_inf."""
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    assert got.shape == want.shape, (got.shape, want.shape)
    scale = max(np.abs(want).max(initial=0.0), 1e-30)
    return float(np.abs(got - want).max(initial=0.0) / scale)


def rel_l2(got, want):
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


def group_scale(name, grads):
    """Analytically-zero tensors (the key-bias gradient, softmax shift invariance)
    are normalised by their layer's QKV-bias group."""
    if name.endswith("key.bias"):
        q = grads.get(name.replace("key.bias", "query.bias"))
        if q is not None:
            return max(np.abs(q).max(), 1e-30)
    return None


def compare_grads(got, want, tol, metric=rel_err):
    worst = (0.0, None)
    assert set(got) == set(want), (sorted(set(got) ^ set(want)))
    for k, w in want.items():
        g = got[k]
        gs = group_scale(k, want)
        if gs is not None:
            e = float(np.abs(np.asarray(g).ravel() - np.asarray(w).ravel()).max() / gs)
        else:
            e = metric(g, w)
        if e > worst[0]:
            worst = (e, k)
    assert worst[0] <= tol, f"worst gradient {worst[1]}: {worst[0]:.3e} > {tol}"
    return worst
