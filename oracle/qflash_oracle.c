/*
 * qflash_oracle.c -- plain, slow, obviously-correct CPU oracle for the QFlash
 * hot path (arxiv 2604.25306).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path (libqflash.so and the
 * paper_2604_25306_b200 package) never links, imports or executes it, and the
 * two share no code: this file derives every constant itself from the paper.
 *
 * Citations: "P:Lnnn" = line nnn of the paper source; R# = the
 * reading of an ambiguous passage recorded in DESIGN.md section "Readings".
 *
 * Arithmetic: int64_t intermediates everywhere (no overflow is possible for the
 * admissible shapes), fp64 for the host-side constants, fp32 IEEE for the
 * quantizer exactly as R2 fixes it.  Floor division is written out explicitly
 * (C's '/' truncates toward zero).
 *
 * Parity pins: every function below is pinned by tests/test_oracle_pins.py to
 * values the paper prints, closed forms, invariants or brute force (see the
 * table in DESIGN.md "Oracle pins").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define QO_OK 0
#define QO_ERR_INVALID 1
#define QO_ERR_SHAPE 2
#define QO_ERR_SCALE 3

/* log2(e) literal (Alg. 1 Require). */
#define QO_LOG2E 1.4426950408889634

/* ---------------------------------------------------------------- helpers */

/* floor(a / b) for b > 0 (mathematical floor, unlike C's truncation). */
int64_t qo_floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && (a < 0)) q -= 1;
  return q;
}

/* round-half-away-from-zero of a double (R1: the paper's rounding |.] ). */
static double qo_round(double x) { return round(x); }

/* ------------------------------------------------ Eq. 1-2: quantization */

/* Eq. 2: s_X = ||X||_inf / (2^(b-1)-1), X^ = round(X / s_X), b=8.
 * R2: fp32 arithmetic, IEEE division, roundf (half away).  R3: a tensor whose
 * scale is zero -- all-zero, or so small (amax <= 127 * 2^-150) that fl32(amax/127)
 * underflows -- gets s = 1/127 (Eq. 2 divides by s).  R4: saturate to
 * [-128, 127] (Eq. 1). */
static float qo_scale_from_amax(float amax) {
  const float s = amax / 127.0f;
  if (s == 0.0f) return 1.0f / 127.0f;
  return s;
}

static int8_t qo_quantize_one(float x, float s) {
  float t = roundf(x / s);
  if (t > 127.0f) t = 127.0f;
  if (t < -128.0f) t = -128.0f;
  return (int8_t)t;
}

int qo_quantize_f32(const float* x, int64_t n, int8_t* xq, float* scale_out) {
  if (!x || !xq || !scale_out || n < 0) return QO_ERR_INVALID;
  float amax = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    float a = fabsf(x[i]);
    if (a > amax) amax = a;
  }
  float s = qo_scale_from_amax(amax);
  for (int64_t i = 0; i < n; ++i) xq[i] = qo_quantize_one(x[i], s);
  *scale_out = s;
  return QO_OK;
}

/* bf16 input: widened exactly to fp32 (bf16 is the top half of an fp32). */
int qo_quantize_bf16(const uint16_t* x, int64_t n, int8_t* xq, float* scale_out) {
  if (!x || !xq || !scale_out || n < 0) return QO_ERR_INVALID;
  float* w = (float*)malloc((size_t)(n > 0 ? n : 1) * sizeof(float));
  if (!w) return QO_ERR_INVALID;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t bits = ((uint32_t)x[i]) << 16;
    memcpy(&w[i], &bits, 4);
  }
  int rc = qo_quantize_f32(w, n, xq, scale_out);
  free(w);
  return rc;
}

/* Inverse of Eq. 2: y = s * x^ in fp32. */
void qo_dequantize(const int8_t* xq, int64_t n, float s, float* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = s * (float)xq[i];
}

/* ------------------------------------------ host-side constants (D6, R6-R8) */

typedef struct {
  double s;      /* s = s_Q * s_K * d^(-1/2) * log2(e)        */
  int64_t s_inv; /* round(1/s)                                (Alg. 2) */
  int32_t n;     /* floor(log2(s / s_P)), s_P = 1/127         (Eq. 9, R8)      */
  int32_t r_p;   /* r = b - n, b = 8                          (Eq. 9)          */
  int64_t m_p;   /* M_r = round((s / s_P) * 2^r)              (Eq. 10)         */
} qo_params;

/* Eq. 9-10: fixed-point multiplier for a real ratio s_X/s_Y:
 *   n = floor(log2(ratio)),  r = b - n,  M_r = round(ratio * 2^r).
 * floor(log2) is taken exactly from the binary exponent (frexp). */
int qo_make_multiplier(double ratio, int32_t b, int32_t* n_out, int32_t* r_out, int64_t* m_out) {
  if (!(ratio > 0.0) || !isfinite(ratio)) return QO_ERR_SCALE;
  int e = 0;
  (void)frexp(ratio, &e); /* ratio = f * 2^e, f in [0.5, 1) => floor(log2) = e-1 */
  const int32_t n = e - 1;
  const int32_t r = b - n;
  *n_out = n;
  *r_out = r;
  *m_out = (int64_t)qo_round(ldexp(ratio, r));
  return QO_OK;
}

/* Returns QO_ERR_SCALE unless 2^-24 <= s <= 0.5 (range in which int64 and the
 * shape bounds keep every step exact; DESIGN.md "Readings" R6). */
int qo_derive_params(float s_q, float s_k, int32_t d, qo_params* out) {
  if (!out) return QO_ERR_INVALID;
  if (d <= 0) return QO_ERR_SHAPE;
  if (!(s_q > 0.0f) || !(s_k > 0.0f) || !isfinite(s_q) || !isfinite(s_k))
    return QO_ERR_SCALE;
  double s = ((double)s_q * (double)s_k) * QO_LOG2E / sqrt((double)d);
  if (!(s >= ldexp(1.0, -24)) || !(s <= 0.5)) return QO_ERR_SCALE;
  out->s = s;
  out->s_inv = (int64_t)qo_round(1.0 / s);
  /* Eq. 9 with s_X = s (ShiftExp2 output scale, Alg. 2 line s_y <- s_x) and
   * s_Y = 1/127 (R8): ratio = s / (1/127) = 127 s, b = 8. */
  return qo_make_multiplier(s * 127.0, 8, &out->n, &out->r_p, &out->m_p);
}

/* ------------------------------------------------ Alg. 2: ShiftExp2 (C2) */

/* eq:q_div: q = floor(x / (-s_inv)), x <= 0.  R6: the oracle
 * defines q by this division; the mul+shift of eq:q_mulshift is the kernel's
 * way of computing the same q faster. */
int64_t qo_quotient_div(int64_t x, int64_t s_inv) {
  return qo_floordiv(-x, s_inv);
}

/* Algorithm 2, x <= 0:
 *   q = floor(x / -s_inv)                     (eq:q_div, R6)
 *   r = x + q * s_inv                         in (-s_inv, 0]
 *   y = ((r >> 1) + s_inv) >> q               arithmetic shifts (floor)
 * R7: a shift by q >= 63 is not evaluated in C; the mathematical floor of a
 * value in [0, s_inv] divided by 2^q is 0 there. */
int64_t qo_shift_exp2(int64_t x, int64_t s_inv) {
  int64_t q = qo_quotient_div(x, s_inv);
  int64_t r = x + q * s_inv;
  int64_t t = qo_floordiv(r, 2) + s_inv; /* (r >> 1) + s_inv */
  if (q >= 62) return 0;
  return qo_floordiv(t, (int64_t)1 << q); /* t >> q */
}

/* Vector form of Algorithm 2 for exhaustive sweeps in the tests. */
void qo_shift_exp2_array(const int64_t* x, int64_t n, int64_t s_inv, int64_t* y) {
  for (int64_t i = 0; i < n; ++i) y[i] = qo_shift_exp2(x[i], s_inv);
}

/* ------------------------------------------------ Eq. 9-10: requantization */

/* Eq. 10: Y = (X * M_r) >> r, then R8 clamp to 127 (P^ in [0,127]). */
int64_t qo_requantize(int64_t y, int64_t m_p, int32_t r_p) {
  int64_t prod = y * m_p;
  int64_t v = (r_p >= 0) ? qo_floordiv(prod, (int64_t)1 << r_p) : prod * ((int64_t)1 << (-r_p));
  if (v > 127) v = 127;
  if (v < -128) v = -128;
  return v;
}

/* ----------------------------------------- Eq. 14 / P:L408: ScaleRelease */

/* R10: floor(X * alpha * s_alpha) realised as floor(X * alpha / s_inv), the
 * "inverse scale approximated as an integer to perform division" of P:L408. */
int64_t qo_scale_release(int64_t x, int64_t alpha, int64_t s_inv) {
  return qo_floordiv(x * alpha, s_inv);
}

/* Step (11): floor(O / l), R14 saturation to int8. */
int64_t qo_normalize(int64_t o, int64_t l) {
  int64_t v = qo_floordiv(o, l);
  if (v > 127) v = 127;
  if (v < -128) v = -128;
  return v;
}

/* -------------------------------------------------- Alg. 1: QFlash forward */

typedef struct {
  const int8_t *q, *k, *v;
  int8_t* out;
  int64_t p_begin, p_end;
  int32_t row_begin, row_end; /* query rows of each problem to compute */
  int32_t N, d, block_r, block_kv, mode;
  qo_params prm;
  int32_t overflow; /* set when mode 1 (scale accumulation) leaves int64 */
  int64_t* l_state; /* optional: final l per computed row (tests only) */
  int64_t* o_state; /* optional: final O per computed row, [rows][d] */
} qo_job;

/* One attention problem p (Algorithm 1).  Q,K,V,O are [N][d].
 * mode 0: Scale Release (Eq. 14, the paper's method);
 * mode 1: Scale Accumulation (Eq. 13, the rejected alternative of App. B.1),
 *         l and O keep the growing scale; PV is divided by s_alpha = s, i.e.
 *         multiplied by s_inv -- reported for the C1 experiment only. */
static void qo_attention_problem(qo_job* jb, int64_t p) {
  const int32_t N = jb->N, d = jb->d, Br = jb->block_r, Bc = jb->block_kv;
  const int64_t s_inv = jb->prm.s_inv;
  const int8_t* Q = jb->q + p * (int64_t)N * d;
  const int8_t* K = jb->k + p * (int64_t)N * d;
  const int8_t* V = jb->v + p * (int64_t)N * d;
  int8_t* Out = jb->out + p * (int64_t)N * d;

  int64_t* S = (int64_t*)malloc(sizeof(int64_t) * (size_t)Br * Bc);
  int64_t* Pm = (int64_t*)malloc(sizeof(int64_t) * (size_t)Br * Bc);
  int64_t* O = (int64_t*)malloc(sizeof(int64_t) * (size_t)Br * d);
  int64_t* m = (int64_t*)malloc(sizeof(int64_t) * (size_t)Br);
  int64_t* l = (int64_t*)malloc(sizeof(int64_t) * (size_t)Br);

  /* Line "Divide Q into T_r = ceil(N/B_r) blocks"; ragged last block.
   * (row_begin/row_end select a sub-range of independent rows; default 0..N.) */
  for (int32_t i0 = jb->row_begin; i0 < jb->row_end; i0 += Br) {
    const int32_t rows = (jb->row_end - i0 < Br) ? (jb->row_end - i0) : Br;
    /* Line "initialize O_i = 0, l_i = 0, m_i = -2^21". */
    for (int32_t a = 0; a < rows; ++a) {
      m[a] = -((int64_t)1 << 21);
      l[a] = 0;
      for (int32_t k = 0; k < d; ++k) O[(int64_t)a * d + k] = 0;
    }
    /* "for j = 1 to T_c", ascending (R17); ragged last tile (R16). */
    for (int32_t j0 = 0; j0 < N; j0 += Bc) {
      const int32_t cols = (N - j0 < Bc) ? (N - j0) : Bc;
      for (int32_t a = 0; a < rows; ++a) {
        const int8_t* qrow = Q + (int64_t)(i0 + a) * d;
        /* (1) S = Q_i K_j^T, exact int32 (Eq. 3). */
        for (int32_t c = 0; c < cols; ++c) {
          const int8_t* krow = K + (int64_t)(j0 + c) * d;
          int64_t acc = 0;
          for (int32_t k = 0; k < d; ++k) acc += (int64_t)qrow[k] * (int64_t)krow[k];
          S[(int64_t)a * Bc + c] = acc;
        }
        /* (2)(3) m_new = max(m_old, rowmax(S)) (Eq. 4). */
        int64_t m_new = m[a];
        for (int32_t c = 0; c < cols; ++c)
          if (S[(int64_t)a * Bc + c] > m_new) m_new = S[(int64_t)a * Bc + c];
        /* (4) alpha = ShiftExp2(m_old - m_new). */
        const int64_t alpha = qo_shift_exp2(m[a] - m_new, s_inv);
        /* (5)(6) P = Requant(ShiftExp2(S - m_new)). */
        int64_t rowsum = 0;
        for (int32_t c = 0; c < cols; ++c) {
          int64_t y = qo_shift_exp2(S[(int64_t)a * Bc + c] - m_new, s_inv);
          int64_t pv = qo_requantize(y, jb->prm.m_p, jb->prm.r_p);
          Pm[(int64_t)a * Bc + c] = pv;
          rowsum += pv; /* (7) Eq. 11 */
        }
        if (jb->mode == 0) {
          /* (7)(9) l = ScaleRelease(l, alpha) + rowsum(P) (Eq. 14). */
          l[a] = qo_scale_release(l[a], alpha, s_inv) + rowsum;
          /* (8)(10) O = ScaleRelease(O, alpha) + P V_j (Eq. 14). */
          for (int32_t k = 0; k < d; ++k) {
            int64_t pv = 0;
            for (int32_t c = 0; c < cols; ++c)
              pv += Pm[(int64_t)a * Bc + c] * (int64_t)V[(int64_t)(j0 + c) * d + k];
            O[(int64_t)a * d + k] = qo_scale_release(O[(int64_t)a * d + k], alpha, s_inv) + pv;
          }
        } else {
          /* Eq. 13: O = O * alpha + floor(PV / s_alpha), s_alpha = s  =>
           * floor(PV / s) realised as PV * s_inv (integer inverse scale,
           * P:L408).  Overflow of int64 is detected, not wrapped (App. B.1). */
          __int128 lw = (__int128)l[a] * alpha + (__int128)rowsum * s_inv;
          if (lw > INT64_MAX || lw < INT64_MIN) jb->overflow = 1;
          l[a] = (int64_t)lw;
          for (int32_t k = 0; k < d; ++k) {
            int64_t pv = 0;
            for (int32_t c = 0; c < cols; ++c)
              pv += Pm[(int64_t)a * Bc + c] * (int64_t)V[(int64_t)(j0 + c) * d + k];
            __int128 ow = (__int128)O[(int64_t)a * d + k] * alpha + (__int128)pv * s_inv;
            if (ow > INT64_MAX || ow < INT64_MIN) jb->overflow = 1;
            O[(int64_t)a * d + k] = (int64_t)ow;
          }
        }
        m[a] = m_new;
      }
    }
    /* (11) O_i = floor(O / l); R14 saturate to int8; s_O = s_V. */
    for (int32_t a = 0; a < rows; ++a) {
      const int32_t row = i0 + a - jb->row_begin;
      if (jb->l_state) jb->l_state[row] = l[a];
      for (int32_t k = 0; k < d; ++k) {
        if (jb->o_state) jb->o_state[(int64_t)row * d + k] = O[(int64_t)a * d + k];
        int64_t o = (l[a] > 0) ? qo_normalize(O[(int64_t)a * d + k], l[a]) : 0;
        Out[(int64_t)(i0 + a) * d + k] = (int8_t)o;
      }
    }
  }
  free(S);
  free(Pm);
  free(O);
  free(m);
  free(l);
}

static void* qo_worker(void* arg) {
  qo_job* jb = (qo_job*)arg;
  for (int64_t p = jb->p_begin; p < jb->p_end; ++p) qo_attention_problem(jb, p);
  return NULL;
}

/* Algorithm 1 over P independent problems ([P][N][d] int8, row-major).
 * block_r only regroups independent rows and cannot change results;
 * block_kv (B_c) is part of the numerical contract (R15).  nthreads > 1 splits
 * the independent problems over pthreads (same per-problem code).
 * Returns QO_OK, QO_ERR_* ; *overflow (may be NULL) reports mode-1 overflow. */
int qo_attention_mode(const int8_t* q, const int8_t* k, const int8_t* v, int64_t P,
                      int32_t N, int32_t d, int32_t block_r, int32_t block_kv, float s_q,
                      float s_k, int32_t mode, int32_t nthreads, int8_t* out,
                      int32_t* overflow) {
  if (!q || !k || !v || !out || P < 0) return QO_ERR_INVALID;
  if (N < 1 || d < 1 || d > 128 || block_r < 1 || block_kv < 1) return QO_ERR_SHAPE;
  qo_params prm;
  int rc = qo_derive_params(s_q, s_k, d, &prm);
  if (rc != QO_OK) return rc;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > P) nthreads = (int32_t)(P > 0 ? P : 1);
  qo_job* jobs = (qo_job*)calloc((size_t)nthreads, sizeof(qo_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int32_t t = 0; t < nthreads; ++t) {
    qo_job* jb = &jobs[t];
    jb->q = q; jb->k = k; jb->v = v; jb->out = out;
    jb->p_begin = P * t / nthreads;
    jb->p_end = P * (t + 1) / nthreads;
    jb->N = N; jb->d = d; jb->block_r = block_r; jb->block_kv = block_kv;
    jb->row_begin = 0; jb->row_end = N;
    jb->mode = mode; jb->prm = prm; jb->overflow = 0;
  }
  if (nthreads == 1) {
    qo_worker(&jobs[0]);
  } else {
    for (int32_t t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, qo_worker, &jobs[t]);
    for (int32_t t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  int32_t ovf = 0;
  for (int32_t t = 0; t < nthreads; ++t) ovf |= jobs[t].overflow;
  if (overflow) *overflow = ovf;
  free(jobs);
  free(th);
  return QO_OK;
}

/* The paper's method (Scale Release), B_r = 128. */
int qo_attention(const int8_t* q, const int8_t* k, const int8_t* v, int64_t P, int32_t N,
                 int32_t d, int32_t block_kv, float s_q, float s_k, int32_t nthreads,
                 int8_t* out) {
  return qo_attention_mode(q, k, v, P, N, d, 128, block_kv, s_q, s_k, 0, nthreads, out, NULL);
}

/* Rows [row_begin, row_end) of problem p computed alone (sampled parity at
 * full size, where the oracle cannot afford every row).  Rows are independent
 * in Algorithm 1 (the outer loop over i), so this is the same
 * arithmetic as qo_attention restricted to those rows.  out_rows receives
 * (row_end - row_begin) * d int8 values. */
int qo_attention_rows_state(const int8_t* q, const int8_t* k, const int8_t* v, int32_t N,
                            int32_t d, int32_t block_kv, float s_q, float s_k, int64_t p,
                            int32_t row_begin, int32_t row_end, int8_t* out_rows,
                            int64_t* l_state, int64_t* o_state) {
  if (!q || !k || !v || !out_rows) return QO_ERR_INVALID;
  if (row_begin < 0 || row_end > N || row_begin >= row_end) return QO_ERR_INVALID;
  if (N < 1 || d < 1 || d > 128 || block_kv < 1) return QO_ERR_SHAPE;
  qo_params prm;
  int rc = qo_derive_params(s_q, s_k, d, &prm);
  if (rc != QO_OK) return rc;
  int8_t* tmp = (int8_t*)malloc((size_t)N * d);
  qo_job jb;
  memset(&jb, 0, sizeof(jb));
  jb.q = q + p * (int64_t)N * d; jb.k = k + p * (int64_t)N * d; jb.v = v + p * (int64_t)N * d;
  jb.out = tmp;
  jb.N = N; jb.d = d; jb.block_r = 128; jb.block_kv = block_kv;
  jb.row_begin = row_begin; jb.row_end = row_end;
  jb.mode = 0; jb.prm = prm;
  jb.l_state = l_state; jb.o_state = o_state;
  qo_attention_problem(&jb, 0);
  memcpy(out_rows, tmp + (int64_t)row_begin * d, (size_t)(row_end - row_begin) * d);
  free(tmp);
  return QO_OK;
}

int qo_attention_rows(const int8_t* q, const int8_t* k, const int8_t* v, int32_t N, int32_t d,
                      int32_t block_kv, float s_q, float s_k, int64_t p, int32_t row_begin,
                      int32_t row_end, int8_t* out_rows) {
  return qo_attention_rows_state(q, k, v, N, d, block_kv, s_q, s_k, p, row_begin, row_end,
                                 out_rows, NULL, NULL);
}
