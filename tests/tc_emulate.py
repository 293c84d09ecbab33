"""Tensor-core emulation for the parity tests (test infrastructure only).

The tcgen05 variants (math "tf32" / "3xtf32") cannot reproduce the
reference interpreter's per-step fp32 chain (interpreter.cc:218-233), so
their parity is stated against an emulation of exactly what the kernels
feed the tensor cores, accumulated in fp64:

  tf32    the MMA reads fp32 operands straight from shared memory and uses
          their top 19 bits (the low 13 mantissa bits are ignored, i.e.
          round toward zero); product sums in fp64.
  3xtf32  hi = the top 19 bits of x (rz: what the MMA itself takes from a
          raw fp32 operand, so the kernels may feed x as hi), lo =
          cvt.rna.tf32(x - hi) (sm100.cuh rzTf32 / toTf32); the kernels
          issue lo*hi + hi*lo + hi*hi into one fp32 accumulator
          (tc_gemm.cu); lo*lo is dropped. Product sums in fp64.

What separates a kernel's output from the emulation is then only the fp32
rounding of the accumulator (~K * 2^-24 of the partial-sum magnitude per MMA
issued per k: one for tf32, three for 3xtf32), so the bound `tol_emu` is four
orders of magnitude tighter than the operand-rounding bound K * 2^-11 it replaces: a
kernel that dropped one 32-deep k-block (~0.1 relative at K = 1024) fails it
by three orders of magnitude (test_emulation_catches_dropped_kblock).
"""
import numpy as np


def tf32_rz(x):
    b = np.ascontiguousarray(x, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32)


def tf32_rna(x):
    """cvt.rna.tf32.f32: round to nearest on the 13 dropped bits, ties away
    from zero (sign-magnitude: add half an ulp to the magnitude, truncate)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32)
    r = (b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)
    return r.view(np.float32)


def split3(x):
    x = np.asarray(x, np.float32)
    hi = tf32_rz(x)
    lo = tf32_rna((x - hi).astype(np.float32))  # x - hi is exact in fp32
    return hi.astype(np.float64), lo.astype(np.float64)


def gemm_nt(A, B, math):
    """sum_k A[.., m, k] * B[.., n, k] as the tensor cores form it (fp64 sums)."""
    if math == "tf32":
        a, b = tf32_rz(A).astype(np.float64), tf32_rz(B).astype(np.float64)
        return np.matmul(a, np.swapaxes(b, -1, -2))
    if math == "3xtf32":
        ah, al = split3(A)
        bh, bl = split3(B)
        bt = lambda t: np.swapaxes(t, -1, -2)  # noqa: E731
        return np.matmul(al, bt(bh)) + np.matmul(ah, bt(bl)) + np.matmul(ah, bt(bh))
    raise ValueError(math)


def fc_relu(I, W, bias, math):
    return np.maximum(bias.astype(np.float64) + gemm_nt(I, W, math), 0.0)


def tol_emu(K, scale=1.0, math="tf32"):
    """Bound on max|got - emu| / max(|emu|, 1) for a K-deep fp32-accumulated
    tensor-core reduction of operands with max|a| * max|b| = scale: K * 2^-24
    per MMA issued into the accumulator for each k (3xtf32 issues three:
    lo*hi, hi*lo, hi*hi)."""
    return (3 if math == "3xtf32" else 1) * K * 2.0 ** -24 * max(1.0, scale)


def gconv_points(I, W1, Bv, idx, math):
    """Emulated tensor-core gconv at flat output indices idx: the implicit
    GEMM over K = C*KH*KW with operands as the kernels round them, plus the
    bias sum (folded into one constant in tensor-core math)."""
    N, G, C, H, W = I.shape
    _, F, _, KH, KW = W1.shape
    Ho, Wo = H - KH + 1, W - KW + 1
    idx = np.asarray(idx, np.int64)
    w = idx % Wo
    r = idx // Wo
    h = r % Ho
    r //= Ho
    o = r % F
    r //= F
    g = r % G
    n = r // G
    if math == "tf32":
        Ia, Wa = tf32_rz(I).astype(np.float64), tf32_rz(W1).astype(np.float64)
        pairs = [(Ia, Wa)]
    else:
        Ih, Il = split3(I)
        Wh, Wl = split3(W1)
        pairs = [(Il, Wh), (Ih, Wl), (Ih, Wh)]
    acc = np.zeros(idx.shape, np.float64)
    for a, b in pairs:
        for kh in range(KH):
            for kw in range(KW):
                patch = a[n, g, :, h + kh, w + kw]       # [P, C]
                filt = b[g, o, :, kh, kw]                # [P, C]
                acc += np.sum(patch * filt, axis=1)
    return acc + float(np.sum(Bv.astype(np.float64)))
