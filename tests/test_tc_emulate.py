"""CPU checks of the tensor-core emulation the tcgen05 parity tests use
(tests/tc_emulate.py): the rounding helpers, and that its tight bound has
teeth — a result missing one 32-deep k-block fails it by orders of
magnitude, while the operand-rounding bound it replaced (K * 2^-11) would
have let that through."""
import numpy as np

import tc_emulate as emu
from conftest import max_rel


def test_tf32_rounding_modes():
    x = np.array([1.0, 1.0 + 2 ** -11, 1.0 + 2 ** -10 + 2 ** -11, -1.0 - 2 ** -11, 1.0 + 3 * 2 ** -12,
                  1.0 + 2 ** -12, 3.0e-39], np.float32)
    rz = emu.tf32_rz(x)
    rna = emu.tf32_rna(x)
    # truncation keeps 10 explicit mantissa bits
    assert rz[1] == 1.0 and rz[2] == np.float32(1.0 + 2 ** -10)
    # ties go away from zero, both signs
    assert rna[1] == np.float32(1.0 + 2 ** -10)
    assert rna[3] == np.float32(-1.0 - 2 ** -10)
    assert rna[2] == np.float32(1.0 + 2 ** -9)
    assert rna[4] == np.float32(1.0 + 2 ** -10) and rna[5] == 1.0
    for v in (rz, rna):
        assert np.all((v.view(np.uint32) & 0x1FFF) == 0)


def test_split3_is_exact_to_2_22():
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, 10000).astype(np.float32)
    hi, lo = emu.split3(x)
    assert np.all(np.abs(hi + lo - x.astype(np.float64)) <= np.abs(x) * 2.0 ** -21)


def test_emulation_close_to_exact():
    rng = np.random.default_rng(1)
    A = rng.uniform(-1, 1, (64, 1024)).astype(np.float32)
    B = rng.uniform(-1, 1, (48, 1024)).astype(np.float32)
    exact = A.astype(np.float64) @ B.astype(np.float64).T
    assert max_rel(exact, emu.gemm_nt(A, B, "3xtf32")) < 1e-5  # lo*lo dropped: ~2^-22 per product
    assert max_rel(exact, emu.gemm_nt(A, B, "tf32")) < 1024 * 2.0 ** -11


def test_emulation_catches_dropped_kblock():
    rng = np.random.default_rng(2)
    K = 1024
    A = rng.uniform(-1, 1, (128, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (100, K)).astype(np.float32)
    for math in ("tf32", "3xtf32"):
        ref = emu.gemm_nt(A, B, math)
        # an fp32-accumulated result (what a correct kernel produces)
        good = ref.astype(np.float32)
        assert max_rel(ref, good) <= emu.tol_emu(K, math=math)
        # one 32-deep k-block missing
        bad = (ref - emu.gemm_nt(A[:, 256:288], B[:, 256:288], math)).astype(np.float32)
        e = max_rel(ref, bad)
        assert e > 100 * emu.tol_emu(K, math=math), (math, e)
        # a k-block whose products are scaled by (1 + 2^-8) (e.g. a wrong
        # descriptor offset reading a neighbouring, nearly equal value) slips
        # under the old operand-rounding bound K * 2^-11, not under tol_emu
        bad = (ref + 2.0 ** -8 * emu.gemm_nt(A[:, 256:288], B[:, 256:288], math)).astype(np.float32)
        e = max_rel(ref, bad)
        assert emu.tol_emu(K, math=math) < e < K * 2.0 ** -11, (math, e)
