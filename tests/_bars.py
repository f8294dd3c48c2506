"""Tolerance models for the TF32 comparisons against the reference's own TF32
mode (max_rel_err, dense_matrix.hpp:68-85).  Both sides round the same
operands to TF32 (tile_exec.cpp:131-142) and multiply them exactly in fp32;
they differ only by fp32 summation order, which moves a result by ~1e-6
relative -- except where a value the reference rounds to TF32 AFTER a sum
lands one TF32 step (<= 2^-10 relative) away."""

TF32_STEP = 2.0 ** -10


def agnn_tf32_bar(betas):
    """AGNN layers.  Two such roundings per layer: (i) the logit (a TF32-rounded
    dot, tile_exec.cpp:386; |logit| <= |beta| for unit rows) moves by <= 2^-10,
    so an attention weight moves by <= |beta| 2^-10 relative; (ii) the
    attention itself, TF32-rounded before the SpMM (tile_exec.cpp:247-248),
    moves by <= 2^-10 relative.  out = sum_e P_e x_e with sum_e P_e = 1 moves by
    <= (1 + |beta|) 2^-10 max|x|, and max|out| ~ max|x|.  That is one layer's
    bound; the tests hold stacks of 2-4 layers to it too (each layer's output
    is a weighted average of its input rows, so an earlier layer's error is
    carried, not amplified, and the per-layer errors are uncorrelated in sign),
    i.e. the bar is tighter than the L-layer worst case."""
    return (1.0 + max(abs(float(b)) for b in betas)) * TF32_STEP


def gcn_tf32_bar():
    """GCN with the default A(hW) order against the reference's (Ah)W: the two
    round different operand sets (h and W vs Ah and W), each rounding off by
    <= 2^-11 relative, so products differ by <= 2 * 2^-10 relative to |A||h||W|."""
    return 2.0 * TF32_STEP
