/*
 * oracle.h — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference
 * interpreter for the paper benchmark operators of arXiv 1802.04730.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the CPU baseline. The product (paper_1802_04730_b200) never links it.
 *
 * Semantics restated from the reference oracle
 *   backend::interpretReference   proj/src/backend/interpreter.cc:301-349
 *   executeStmtInstance/combine   proj/src/backend/interpreter.cc:218-233, 58-71
 *   TensorData::store (narrowing) proj/src/backend/tensor_data.cc:101-107
 *   `op=!` desugaring             proj/src/sem/specialize.cc:118-138
 * Every update step is `acc = (float)((double)acc + (double)a * (double)b)`:
 * the interpreter widens loads to double, combines in double and narrows to
 * float32 on every store. Loops run in canonical order (LHS iterators outer,
 * reduction iterators inner, first-use order; proj/src/lang/validate.cc:150-194).
 *
 * Parity pinning: outputs of this restatement are compared bit-for-bit with
 * the reference interpreter itself (oracle/_ref, built from the reference
 * sources by oracle/Makefile) on the golden cases in tests/golden/.
 */
#ifndef TCB_ORACLE_H
#define TCB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- deterministic inputs (reference: fillUniform tensor_data.cc:191-209,
 *      makeSessionInputs genetic.cc:255-291; std::mt19937_64 + libstdc++
 *      uniform_real_distribution<double> / uniform_int_distribution<int64_t>) */
typedef struct orc_rng orc_rng;
orc_rng* orc_rng_new(uint64_t seed);
void orc_rng_free(orc_rng* r);
uint64_t orc_rng_next(orc_rng* r);
void orc_rng_fill_f32(orc_rng* r, float* out, int64_t n, double lo, double hi);
void orc_rng_fill_i32(orc_rng* r, int32_t* out, int64_t n, double lo, double hi);

/* FNV-1a 64 over bytes (diagnostics.h:110-122) */
uint64_t orc_fnv1a64(const void* data, int64_t n);

/* ---- operators (each cites its TC source) ---- */

/* tbmm.tc:2-4 / tmm.tc:2-4 (B=1) / C3 PAPER.md:3035 (accumulate=1):
 *   Z(b,n,k) (+)=(!) X(b,n,m) * Y(b,k,m)
 * X[B][N][M], Y[B][K][M], Z[B][N][K]. accumulate=0 → `+=!` (zero init),
 * accumulate=1 → plain `+=` onto the incoming Z (interpreter.cc:235-255). */
void orc_tbmm(const float* X, const float* Y, float* Z, int64_t B, int64_t N,
              int64_t M, int64_t K, int accumulate);

/* mlp1.tc:2-6 (one FC+ReLU layer):
 *   O(b,n) = bias(n); O(b,n) += I(b,m) * W(n,m); O(b,n) = fmaxf(O(b,n), 0)
 * I[B][ldi] (first `Kred` columns used), W[Nout][ldw], O[B][Nout]. */
void orc_fc_relu(const float* I, int64_t ldi, const float* W, int64_t ldw,
                 const float* bias, float* O, int64_t B, int64_t Nout,
                 int64_t Kred);

/* 3KRU PAPER.md:2902-2907:
 *   XW2(m,n0,n1,d2) +=! X(m,n0,n1,r2) * W2(d2,r2)
 *   XW1(m,n0,d1,d2) +=! XW2(m,n0,r1,d2) * W1(d1,r1)
 *   Y(m,d0,d1,d2)   +=! XW1(m,r0,d1,d2) * W0(d0,r0) */
void orc_kru3(const float* W0, const float* W1, const float* W2, const float* X,
              float* Y, float* XW1, float* XW2, int64_t M, int64_t N0, int64_t N1,
              int64_t N2, int64_t D0, int64_t D1, int64_t D2);

/* gconv.tc:2-7:
 *   O(n,g,o,h,w) +=! I(n,g,i,h+kh,w+kw) * W1(g,o,i,kh,kw)
 *   O(n,g,o,h,w)  =  O(n,g,o,h,w) + B(m)          (m = 0..Mb-1, sequential)
 * I[N][G][C][H][W], W1[G][F][C][KH][KW], B[Mb], O[N][G][F][H-KH+1][W-KW+1]. */
void orc_gconv(const float* I, const float* W1, const float* Bv, float* O,
               int64_t N, int64_t G, int64_t C, int64_t H, int64_t W, int64_t F,
               int64_t KH, int64_t KW, int64_t Mb);
/* same arithmetic, evaluated only at the given linear output indices */
void orc_gconv_points(const float* I, const float* W1, const float* Bv,
                      const int64_t* idx, int64_t npts, float* out, int64_t N,
                      int64_t G, int64_t C, int64_t H, int64_t W, int64_t F,
                      int64_t KH, int64_t KW, int64_t Mb);

/* 2lut.tc:2-6 (one of the two tables):
 *   O(i,j) +=! LUT(I(i,k), j)
 * LUT[E][D], I[B][L] int32, O[B][D]. Returns 0, or -1 on an index outside
 * [0,E) (IndexOutOfRange, interpreter.cc:284-292). */
int orc_lut(const float* LUT, int64_t E, int64_t D, const int32_t* I, int64_t B,
            int64_t L, float* O);

/* threads used by the OpenMP loops (0 = runtime default) */
void orc_set_threads(int n);
int orc_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
