"""Documented oracle extension for causal attention.

TEST INFRASTRUCTURE ONLY — nothing in paper_2302_08005_b200/ imports or runs
anything this script produces.

The reference op set has no mask op (proj/src/shape_inference.cpp:10-16), so a
decoder (GPT-Neo, BASELINE.json C4) has no reference semantics. This script
derives a *patched copy* of the reference executor that adds exactly one thing:
an optional integer attr ``causal`` on the ``softmax`` op. With ``causal`` = 1
the softmax over the last axis of a (..., Sq, Sk) tensor only covers keys
k <= q + (Sk - Sq); the excluded probabilities are exactly 0. Everything else
(dropout draws over the full (Sq, Sk) index space, the backward formula
P*(dP - sum(dP*P)), quantisation, tape) is the reference's unchanged code — the
backward needs no change because masked probabilities are 0.

It also forwards a ``causal`` attr of an ``EfficientAttention`` module to the
softmax of its reference graph (proj/src/executor.cpp:503-528), so a scheduled
decoder (replace core with EfficientAttention, attrs copied by
library.cpp:106-113) keeps its mask.

The patched file is written to oracle/_ref/causal/executor.cpp (git-ignored)
and compiled by oracle/Makefile into oracle/_ref/slapo_ref_driver_causal; the
unpatched driver is untouched. Each replacement is anchored on a unique line of
the reference and asserted to match exactly once, so a changed reference fails
loudly instead of silently producing an unpatched oracle.

Sites (proj/src/executor.cpp): softmax_rows :189-202 (helper added after it),
forward softmax op :907-916, backward softmax op :1313-1332, attention
reference graph :519.
"""
import os
import sys

REF = os.environ.get("REF", "/root/reference/proj")

HELPER = r'''
// ---- oracle extension (oracle/causal_ext.py): causal softmax ----
// Row r of a (rows, n) view whose second-to-last extent is nq is query
// q = r % nq; it covers keys [0, min(n, q + 1 + n - nq)); the rest are 0.
void softmax_rows_causal(const double* in, double* out, std::int64_t rows, std::int64_t n, std::int64_t nq) {
    for (std::int64_t r = 0; r < rows; ++r) {
        const double* pi = in + r * n;
        double* po = out + r * n;
        std::int64_t lim = std::min<std::int64_t>(n, r % nq + 1 + (n - nq));
        if (lim < 1) lim = 1;
        double mx = pi[0];
        for (std::int64_t i = 1; i < lim; ++i) mx = std::max(mx, pi[i]);
        double sum = 0.0;
        for (std::int64_t i = 0; i < lim; ++i) {
            po[i] = std::exp(pi[i] - mx);
            sum += po[i];
        }
        for (std::int64_t i = 0; i < lim; ++i) po[i] /= sum;
        for (std::int64_t i = lim; i < n; ++i) po[i] = 0.0;
    }
}
void softmax_rows_ext(const double* in, double* out, std::int64_t rows, std::int64_t n, const TensorSpec& s,
                      bool causal) {
    if (!causal) return softmax_rows(in, out, rows, n);
    if (s.rank() < 2) throw Error("causal softmax needs a rank >= 2 input");
    softmax_rows_causal(in, out, rows, n, s.shape[s.rank() - 2]);
}
'''

# (anchor, replacement) pairs; each anchor must occur exactly once
EDITS = [
    # helper after softmax_rows (ends with the closing brace before the AxisView comment)
    ("/// Move `axis` to the last position so row-wise kernels apply; identity when\n",
     HELPER + "\n/// Move `axis` to the last position so row-wise kernels apply; identity when\n"),
    # forward softmax op
    ("            softmax_rows(view.moved.data.data(), y.data.data(), y.size() / nn, nn);\n",
     "            if (attr_int(n.attrs, \"causal\").value_or(0) && axis != x.spec.rank() - 1)\n"
     "                throw Error(\"causal softmax must run over the last axis\");\n"
     "            softmax_rows_ext(view.moved.data.data(), y.data.data(), y.size() / nn, nn, view.moved.spec,\n"
     "                             attr_int(n.attrs, \"causal\").value_or(0) != 0);\n"),
    # backward softmax op (recomputes y)
    ("            softmax_rows(xv.moved.data.data(), y.data.data(), rows, n);\n",
     "            softmax_rows_ext(xv.moved.data.data(), y.data.data(), rows, n, xv.moved.spec,\n"
     "                             attr_int(rec.attrs, \"causal\").value_or(0) != 0);\n"),
    # EfficientAttention's reference graph keeps the module's causal attr
    ("        int attn = b.call_op(\"softmax\", {scaled}, {{\"axis\", std::int64_t(-1)}});\n",
     "        AttrMap smx{{\"axis\", std::int64_t(-1)}};\n"
     "        if (attr_int(ea.attrs, \"causal\").value_or(0)) smx[\"causal\"] = std::int64_t(1);\n"
     "        int attn = b.call_op(\"softmax\", {scaled}, smx);\n"),
]


def main(out_path: str) -> None:
    src = open(os.path.join(REF, "src", "executor.cpp")).read()
    for anchor, repl in EDITS:
        n = src.count(anchor)
        if n != 1:
            sys.exit(f"causal_ext: anchor matched {n} times (expected 1): {anchor.strip()[:80]}")
        src = src.replace(anchor, repl)
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path + ".tmp", "w") as f:
        f.write("// GENERATED by oracle/causal_ext.py from " + REF + "/src/executor.cpp — do not edit\n")
        f.write(src)
    os.replace(out_path + ".tmp", out_path)


if __name__ == "__main__":
    main(sys.argv[1])
