/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h). CPU restatement of
 * the reference interpreter's arithmetic for the paper operators.
 *
 * The single rule every reduction follows (interpreter.cc:218-233 +
 * tensor_data.cc:101-107): load widens float->double, `combine` adds in
 * double, `store` narrows to float. Plain `=` statements evaluate their
 * RHS in double and narrow once.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* one `+=` step of the interpreter: combine(PlusEq) then narrow on store */
static inline float step_fma(float acc, float a, float b) {
  return (float)((double)acc + (double)a * (double)b);
}
static inline float step_add(float acc, float v) {
  return (float)((double)acc + (double)v);
}
/* `fmaxf` builtin → std::fmax in double (interpreter.cc:22-24) */
static inline float relu_store(float v) {
  return (float)fmax((double)v, 0.0);
}

/* ------------------------------------------------------------------ rng */
/* std::mt19937_64 (w=64 n=312 m=156 r=31), restated. */
#define MT_N 312
#define MT_M 156
struct orc_rng {
  uint64_t mt[MT_N];
  int idx;
};

orc_rng* orc_rng_new(uint64_t seed) {
  orc_rng* r = (orc_rng*)malloc(sizeof(orc_rng));
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
  return r;
}

void orc_rng_free(orc_rng* r) { free(r); }

uint64_t orc_rng_next(orc_rng* r) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t A = 0xB5026F5AA96619E9ULL;
  if (r->idx >= MT_N) {
    int i;
    for (i = 0; i < MT_N - MT_M; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + MT_M] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    for (; i < MT_N - 1; ++i) {
      uint64_t x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
      r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    uint64_t x = (r->mt[MT_N - 1] & UM) | (r->mt[0] & LM);
    r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* generate_canonical<double,53>(mt19937_64): one draw, divided by 2^64 */
static double canonical01(orc_rng* r) {
  double v = (double)orc_rng_next(r) / 18446744073709551616.0;
  if (v >= 1.0) v = nextafter(1.0, 0.0);
  return v;
}

void orc_rng_fill_f32(orc_rng* r, float* out, int64_t n, double lo, double hi) {
  for (int64_t k = 0; k < n; ++k) out[k] = (float)(canonical01(r) * (hi - lo) + lo);
}

/* uniform_int_distribution<int64_t>(ceil(lo), ceil(hi)-1) — libstdc++ uses
 * Lemire's nearly-divisionless downscaling for a 64-bit engine. */
void orc_rng_fill_i32(orc_rng* r, int32_t* out, int64_t n, double lo, double hi) {
  int64_t ilo = (int64_t)ceil(lo);
  int64_t ihi = (int64_t)ceil(hi) - 1;
  uint64_t range = (uint64_t)(ihi - ilo) + 1ULL; /* ≥ 1 */
  for (int64_t k = 0; k < n; ++k) {
    unsigned __int128 prod = (unsigned __int128)orc_rng_next(r) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
      uint64_t threshold = (0ULL - range) % range;
      while (low < threshold) {
        prod = (unsigned __int128)orc_rng_next(r) * range;
        low = (uint64_t)prod;
      }
    }
    out[k] = (int32_t)((int64_t)(uint64_t)(prod >> 64) + ilo);
  }
}

uint64_t orc_fnv1a64(const void* data, int64_t n) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

void orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------ operators */

void orc_tbmm(const float* X, const float* Y, float* Z, int64_t B, int64_t N,
              int64_t M, int64_t K, int accumulate) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < B; ++b)
    for (int64_t n = 0; n < N; ++n) {
      const float* x = X + (b * N + n) * M;
      for (int64_t k = 0; k < K; ++k) {
        const float* y = Y + (b * K + k) * M;
        float* z = Z + (b * N + n) * K + k;
        float acc = accumulate ? *z : 0.0f; /* `+=!` → synthetic 0 store */
        for (int64_t m = 0; m < M; ++m) acc = step_fma(acc, x[m], y[m]);
        *z = acc;
      }
    }
}

void orc_fc_relu(const float* I, int64_t ldi, const float* W, int64_t ldw,
                 const float* bias, float* O, int64_t B, int64_t Nout,
                 int64_t Kred) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t b = 0; b < B; ++b)
    for (int64_t n = 0; n < Nout; ++n) {
      float acc = bias[n];                         /* O(b,n) = B1(n) */
      const float* x = I + b * ldi;
      const float* w = W + n * ldw;
      for (int64_t m = 0; m < Kred; ++m) acc = step_fma(acc, x[m], w[m]);
      O[b * Nout + n] = relu_store(acc);           /* fmaxf(O, 0) */
    }
}

void orc_kru3(const float* W0, const float* W1, const float* W2, const float* X,
              float* Y, float* XW1, float* XW2, int64_t M, int64_t N0, int64_t N1,
              int64_t N2, int64_t D0, int64_t D1, int64_t D2) {
  /* statement 1: XW2(m,n0,n1,d2) +=! X(m,n0,n1,r2) * W2(d2,r2) */
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < M; ++m)
    for (int64_t n0 = 0; n0 < N0; ++n0)
      for (int64_t n1 = 0; n1 < N1; ++n1)
        for (int64_t d2 = 0; d2 < D2; ++d2) {
          float acc = 0.0f;
          const float* x = X + ((m * N0 + n0) * N1 + n1) * N2;
          for (int64_t r2 = 0; r2 < N2; ++r2) acc = step_fma(acc, x[r2], W2[d2 * N2 + r2]);
          XW2[((m * N0 + n0) * N1 + n1) * D2 + d2] = acc;
        }
  /* statement 2: XW1(m,n0,d1,d2) +=! XW2(m,n0,r1,d2) * W1(d1,r1) */
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < M; ++m)
    for (int64_t n0 = 0; n0 < N0; ++n0)
      for (int64_t d1 = 0; d1 < D1; ++d1)
        for (int64_t d2 = 0; d2 < D2; ++d2) {
          float acc = 0.0f;
          for (int64_t r1 = 0; r1 < N1; ++r1)
            acc = step_fma(acc, XW2[((m * N0 + n0) * N1 + r1) * D2 + d2], W1[d1 * N1 + r1]);
          XW1[((m * N0 + n0) * D1 + d1) * D2 + d2] = acc;
        }
  /* statement 3: Y(m,d0,d1,d2) +=! XW1(m,r0,d1,d2) * W0(d0,r0) */
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < M; ++m)
    for (int64_t d0 = 0; d0 < D0; ++d0)
      for (int64_t d1 = 0; d1 < D1; ++d1)
        for (int64_t d2 = 0; d2 < D2; ++d2) {
          float acc = 0.0f;
          for (int64_t r0 = 0; r0 < N0; ++r0)
            acc = step_fma(acc, XW1[((m * N0 + r0) * D1 + d1) * D2 + d2], W0[d0 * N0 + r0]);
          Y[((m * D0 + d0) * D1 + d1) * D2 + d2] = acc;
        }
}

static inline float gconv_one(const float* I, const float* W1, const float* Bv,
                              int64_t n, int64_t g, int64_t o, int64_t h, int64_t w,
                              int64_t G, int64_t C, int64_t H, int64_t W, int64_t F,
                              int64_t KH, int64_t KW, int64_t Mb) {
  float acc = 0.0f;
  for (int64_t i = 0; i < C; ++i)
    for (int64_t kh = 0; kh < KH; ++kh)
      for (int64_t kw = 0; kw < KW; ++kw)
        acc = step_fma(acc, I[(((n * G + g) * C + i) * H + h + kh) * W + w + kw],
                       W1[(((g * F + o) * C + i) * KH + kh) * KW + kw]);
  /* statement 2 repeats `O = O + B(m)` for every m (validate.cc:190-194) */
  for (int64_t m = 0; m < Mb; ++m) acc = step_add(acc, Bv[m]);
  return acc;
}

void orc_gconv(const float* I, const float* W1, const float* Bv, float* O,
               int64_t N, int64_t G, int64_t C, int64_t H, int64_t W, int64_t F,
               int64_t KH, int64_t KW, int64_t Mb) {
  const int64_t Ho = H - KH + 1, Wo = W - KW + 1;
#pragma omp parallel for collapse(3) schedule(static)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t g = 0; g < G; ++g)
      for (int64_t o = 0; o < F; ++o)
        for (int64_t h = 0; h < Ho; ++h)
          for (int64_t w = 0; w < Wo; ++w)
            O[(((n * G + g) * F + o) * Ho + h) * Wo + w] =
                gconv_one(I, W1, Bv, n, g, o, h, w, G, C, H, W, F, KH, KW, Mb);
}

void orc_gconv_points(const float* I, const float* W1, const float* Bv,
                      const int64_t* idx, int64_t npts, float* out, int64_t N,
                      int64_t G, int64_t C, int64_t H, int64_t W, int64_t F,
                      int64_t KH, int64_t KW, int64_t Mb) {
  const int64_t Ho = H - KH + 1, Wo = W - KW + 1;
  (void)N;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < npts; ++p) {
    int64_t r = idx[p];
    int64_t w = r % Wo; r /= Wo;
    int64_t h = r % Ho; r /= Ho;
    int64_t o = r % F; r /= F;
    int64_t g = r % G; r /= G;
    int64_t n = r;
    out[p] = gconv_one(I, W1, Bv, n, g, o, h, w, G, C, H, W, F, KH, KW, Mb);
  }
}

int orc_lut(const float* LUT, int64_t E, int64_t D, const int32_t* I, int64_t B,
            int64_t L, float* O) {
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
  for (int64_t i = 0; i < B; ++i)
    for (int64_t j = 0; j < D; ++j) {
      float acc = 0.0f;
      for (int64_t k = 0; k < L; ++k) {
        int64_t e = (int64_t)I[i * L + k];
        if (e < 0 || e >= E) {
          bad = 1;
          break;
        }
        acc = step_add(acc, LUT[e * D + j]);
      }
      O[i * D + j] = acc;
    }
  return bad ? -1 : 0;
}
