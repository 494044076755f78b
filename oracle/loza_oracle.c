/*
 * loza_oracle.c — plain, slow, fp64 CPU oracle for the LoZA / SSA hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no code,
 * header, table or constant generator with the CUDA path (paper_2512_23966_b200/),
 * and the CUDA path never loads it.
 *
 * Every function follows a plain definition from the paper, in the paper's order:
 *   - Eq. 1  full attention  O = softmax(QK)V, read with an
 *     explicit scale and K transposed ("details ... omitted";
 *     DESIGN.md reading R1) and a causal mask j <= i (reading R3).
 *   - Eq. 4 SSA O* = softmax(QK*)V*, K*,V* = "anchored and
 *     blocked keys and values (#sink blocks s, #local blocks l, block size b)";
 *     PAPER.md:49 "one query token only attends to several sink and local blocks".
 *     Token-level mask (readings R2-R5):
 *         allowed(i, j) <=> j <= i  and  ( floor(j/b) < s  or  floor(i/b) - floor(j/b) < l )
 *   - Eq. 3 blend  O^ = a*O + (1-a)*O'  and its scalar
 *     gradient dL/da = <dO^, O - O'> (calculus of Eq. 3).
 *
 * No blocking, no fusion, no online softmax: per query row the explicit mask
 * row is materialised over all n_kv keys, the masked logits are skipped, and
 * the softmax is the textbook max-shifted exp / sum, all in double precision.
 * Inputs are fp32 arrays holding the exact values the device consumed (bf16 and
 * fp32 widen exactly).
 *
 * Parity pins (tests/test_oracle_pins.py, none re-types these formulas):
 *   mask / selection   hand example SPEC.md:124, closed-form block counts,
 *                      window = 1024 at (1,7,128), brute-force
 *                      pair counts, dense-causal degeneracy
 *   attention          torch SDPA (fp64 library routine) on the dense-causal and
 *                      explicit-mask cases, O = V closed forms, Q = 0 => mean,
 *                      V = c => O = c, LSE(Q=0) = ln(#allowed), perturbation
 *                      invariance
 *   blend              endpoints, linearity / finite difference
 *
 *   backward           central finite differences of L = sum dO.O through the forward
 *                      oracle (fp64) on q, k, v entries; single key => dq = dk = 0,
 *                      dv = sum dO; constant V => dq = dk = 0
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* allowed(p, j) for one query at absolute position p.
 * sparse = 0 gives full attention (Eq. 1); causal = 0 drops j <= p (full only). */
static int allowed(int64_t p, int64_t j, int32_t s, int32_t l, int32_t b, int32_t sparse,
                   int32_t causal) {
  if (causal && j > p) return 0;
  if (!sparse) return 1;
  {
    const int64_t qblk = p / b, kblk = j / b;
    return (kblk < s) || (qblk - kblk < l);
  }
}

/* Explicit mask row M[j], j in [0, n_kv). */
void loza_oracle_mask_row(int64_t p, int64_t n_kv, int32_t s, int32_t l, int32_t b,
                          int32_t sparse, int32_t causal, uint8_t* out) {
  for (int64_t j = 0; j < n_kv; ++j) out[j] = (uint8_t)allowed(p, j, s, l, b, sparse, causal);
}

/* Positions j with M[j] = 1, ascending; returns the count. */
int64_t loza_oracle_allowed_keys(int64_t p, int64_t n_kv, int32_t s, int32_t l, int32_t b,
                                 int32_t sparse, int32_t causal, int64_t* out_pos) {
  int64_t c = 0;
  uint8_t* m = (uint8_t*)malloc((size_t)(n_kv > 0 ? n_kv : 1));
  loza_oracle_mask_row(p, n_kv, s, l, b, sparse, causal, m);
  for (int64_t j = 0; j < n_kv; ++j)
    if (m[j]) out_pos[c++] = j;
  free(m);
  return c;
}

/* Block selection (SURVEY.md §8 c-i step 5): key block kb is selected for query
 * block QB  <=>  some query i in QB and key j in kb have M_i[j] = 1.
 * Queries are the absolute positions [q_start, q_start + n_q); query block
 * qb_local covers [q_start + qb_local*b, ...) (q_start is a multiple of b).
 * out_idx[qb_local*max_sel + t] ascending absolute key blocks, -1 padded. */
int loza_oracle_select_blocks(int64_t n_q, int64_t q_start, int64_t n_kv, int32_t s, int32_t l,
                              int32_t b, int32_t causal, const int64_t* qb_list, int64_t n_list,
                              int32_t max_sel, int32_t* out_idx, int32_t* out_count) {
  const int64_t n_kb = (n_kv + b - 1) / b;
  int err = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t t = 0; t < n_list; ++t) {
    const int64_t qbl = qb_list[t];
    uint8_t* sel = (uint8_t*)calloc((size_t)(n_kb > 0 ? n_kb : 1), 1);
    uint8_t* m = (uint8_t*)malloc((size_t)(n_kv > 0 ? n_kv : 1));
    const int64_t i0 = q_start + qbl * b;
    int64_t i1 = i0 + b;
    if (i1 > q_start + n_q) i1 = q_start + n_q;
    for (int64_t p = i0; p < i1; ++p) {
      loza_oracle_mask_row(p, n_kv, s, l, b, 1, causal, m);
      for (int64_t j = 0; j < n_kv; ++j)
        if (m[j]) sel[j / b] = 1;
    }
    int32_t c = 0;
    for (int64_t kb = 0; kb < n_kb; ++kb) {
      if (!sel[kb]) continue;
      if (c < max_sel) out_idx[t * max_sel + c] = (int32_t)kb;
      ++c;
    }
    for (int32_t r = c; r < max_sel; ++r) out_idx[t * max_sel + r] = -1;
    if (c > max_sel) {
#pragma omp atomic write
      err = 1;
    }
    out_count[t] = c;
    free(sel);
    free(m);
  }
  return err;
}

/* softmax(scale * q k^T) v over exactly the given key rows (already the allowed
 * set), fp64. q [R][d_qk]; k [nk][d_qk]; v [nk][d_v] (row strides in elements).
 * o [R][d_v]; lse [R] (natural log) may be NULL. */
void loza_oracle_attend(const float* q, int64_t R, int64_t q_stride, const float* k,
                        int64_t k_stride, const float* v, int64_t v_stride, int64_t nk,
                        int32_t d_qk, int32_t d_v, double scale, double* o, double* lse) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < R; ++r) {
    const float* qr = q + r * q_stride;
    double* z = (double*)malloc(sizeof(double) * (size_t)(nk > 0 ? nk : 1));
    double m = -INFINITY;
    for (int64_t j = 0; j < nk; ++j) {
      const float* kj = k + j * k_stride;
      double acc = 0.0;
      for (int32_t d = 0; d < d_qk; ++d) acc += (double)qr[d] * (double)kj[d];
      z[j] = scale * acc;
      if (z[j] > m) m = z[j];
    }
    double L = 0.0;
    for (int64_t j = 0; j < nk; ++j) {
      z[j] = exp(z[j] - m);
      L += z[j];
    }
    double* orow = o + r * d_v;
    for (int32_t d = 0; d < d_v; ++d) orow[d] = 0.0;
    for (int64_t j = 0; j < nk; ++j) {
      const float* vj = v + j * v_stride;
      const double w = z[j];
      for (int32_t d = 0; d < d_v; ++d) orow[d] += w * (double)vj[d];
    }
    for (int32_t d = 0; d < d_v; ++d) orow[d] /= L;
    if (lse) lse[r] = m + log(L);
    free(z);
  }
}

/* Attention for R query rows with absolute positions pos[r] against one full
 * K/V sequence of n_kv rows: materialise the mask row, skip masked keys
 * (identical to exp(-inf) = 0), textbook softmax in fp64. */
void loza_oracle_attention_rows(const float* q, const int64_t* pos, int64_t R, int64_t q_stride,
                                const float* k, int64_t k_stride, const float* v,
                                int64_t v_stride, int64_t n_kv, int32_t d_qk, int32_t d_v,
                                double scale, int32_t s, int32_t l, int32_t b, int32_t sparse,
                                int32_t causal, double* o, double* lse) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < R; ++r) {
    uint8_t* mrow = (uint8_t*)malloc((size_t)(n_kv > 0 ? n_kv : 1));
    double* z = (double*)malloc(sizeof(double) * (size_t)(n_kv > 0 ? n_kv : 1));
    const float* qr = q + r * q_stride;
    loza_oracle_mask_row(pos[r], n_kv, s, l, b, sparse, causal, mrow);
    double m = -INFINITY;
    for (int64_t j = 0; j < n_kv; ++j) {
      if (!mrow[j]) continue;
      const float* kj = k + j * k_stride;
      double acc = 0.0;
      for (int32_t d = 0; d < d_qk; ++d) acc += (double)qr[d] * (double)kj[d];
      z[j] = scale * acc;
      if (z[j] > m) m = z[j];
    }
    double L = 0.0;
    for (int64_t j = 0; j < n_kv; ++j) {
      if (!mrow[j]) continue;
      z[j] = exp(z[j] - m);
      L += z[j];
    }
    double* orow = o + r * d_v;
    for (int32_t d = 0; d < d_v; ++d) orow[d] = 0.0;
    for (int64_t j = 0; j < n_kv; ++j) {
      if (!mrow[j]) continue;
      const float* vj = v + j * v_stride;
      for (int32_t d = 0; d < d_v; ++d) orow[d] += z[j] * (double)vj[d];
    }
    for (int32_t d = 0; d < d_v; ++d) orow[d] /= L;
    if (lse) lse[r] = m + log(L);
    free(mrow);
    free(z);
  }
}

/* Eq. 3 forward and its scalar gradient, fp64, on the exact inputs:
 *   ohat = a*o + (1-a)*op ;  dalpha = sum_e dohat_e * (o_e - op_e).
 * dohat / ohat / dalpha may be NULL. */
void loza_oracle_blend(const float* o, const float* op, double alpha, const float* dohat,
                       int64_t n, double* ohat, double* dalpha) {
  if (ohat) {
#pragma omp parallel for
    for (int64_t e = 0; e < n; ++e) ohat[e] = alpha * (double)o[e] + (1.0 - alpha) * (double)op[e];
  }
  if (dohat && dalpha) {
    double acc = 0.0;
#pragma omp parallel for reduction(+ : acc)
    for (int64_t e = 0; e < n; ++e) acc += (double)dohat[e] * ((double)o[e] - (double)op[e]);
    *dalpha = acc;
  }
}

/* Backward of Eq. 1 / Eq. 4 (softmax attention over the allowed keys), fp64, for R query rows at absolute
 * positions pos[r] against one K/V sequence of n_kv rows. The chain rule of O_r = sum_j P_rj v_j with
 * P_rj = exp(z_rj - m_r) / L_r and z_rj = scale q_r . k_j over the allowed j, for a loss with dL/dO_r = do_r:
 *   dP_rj = do_r . v_j ;  D_r = sum_j P_rj dP_rj (= do_r . O_r) ;  dZ_rj = P_rj (dP_rj - D_r)
 *   dq_r = scale sum_j dZ_rj k_j ;  dk_j = scale sum_r dZ_rj q_r ;  dv_j = sum_r P_rj do_r
 * Pass 1 (rows): m_r, L_r, D_r and dq_r. Pass 2 (keys): dk_j, dv_j over the rows that allow j (no reduction
 * races). dq [R][d_qk], dk [n_kv][d_qk], dv [n_kv][d_v] are written (fp64). */
void loza_oracle_attention_backward(const float* q, const int64_t* pos, int64_t R, int64_t q_stride,
                                    const float* k, int64_t k_stride, const float* v, int64_t v_stride,
                                    const float* dout, int64_t do_stride, int64_t n_kv, int32_t d_qk,
                                    int32_t d_v, double scale, int32_t s, int32_t l, int32_t b,
                                    int32_t sparse, int32_t causal, double* dq, double* dk, double* dv) {
  double* m = (double*)malloc(sizeof(double) * (size_t)(R > 0 ? R : 1));
  double* L = (double*)malloc(sizeof(double) * (size_t)(R > 0 ? R : 1));
  double* D = (double*)malloc(sizeof(double) * (size_t)(R > 0 ? R : 1));
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < R; ++r) {
    uint8_t* mrow = (uint8_t*)malloc((size_t)(n_kv > 0 ? n_kv : 1));
    double* z = (double*)malloc(sizeof(double) * (size_t)(n_kv > 0 ? n_kv : 1));
    const float* qr = q + r * q_stride;
    const float* dor = dout + r * do_stride;
    loza_oracle_mask_row(pos[r], n_kv, s, l, b, sparse, causal, mrow);
    double mx = -INFINITY;
    for (int64_t j = 0; j < n_kv; ++j) {
      if (!mrow[j]) continue;
      const float* kj = k + j * k_stride;
      double acc = 0.0;
      for (int32_t d = 0; d < d_qk; ++d) acc += (double)qr[d] * (double)kj[d];
      z[j] = scale * acc;
      if (z[j] > mx) mx = z[j];
    }
    double Ls = 0.0;
    for (int64_t j = 0; j < n_kv; ++j)
      if (mrow[j]) Ls += exp(z[j] - mx);
    double Dr = 0.0;  /* D_r = sum_j P_rj dP_rj */
    for (int64_t j = 0; j < n_kv; ++j) {
      if (!mrow[j]) continue;
      const float* vj = v + j * v_stride;
      double dp = 0.0;
      for (int32_t d = 0; d < d_v; ++d) dp += (double)dor[d] * (double)vj[d];
      Dr += exp(z[j] - mx) / Ls * dp;
    }
    double* dqr = dq + r * d_qk;
    for (int32_t d = 0; d < d_qk; ++d) dqr[d] = 0.0;
    for (int64_t j = 0; j < n_kv; ++j) {
      if (!mrow[j]) continue;
      const float* vj = v + j * v_stride;
      const float* kj = k + j * k_stride;
      double dp = 0.0;
      for (int32_t d = 0; d < d_v; ++d) dp += (double)dor[d] * (double)vj[d];
      const double dz = exp(z[j] - mx) / Ls * (dp - Dr);
      for (int32_t d = 0; d < d_qk; ++d) dqr[d] += scale * dz * (double)kj[d];
    }
    m[r] = mx;
    L[r] = Ls;
    D[r] = Dr;
    free(mrow);
    free(z);
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t j = 0; j < n_kv; ++j) {
    const float* kj = k + j * k_stride;
    const float* vj = v + j * v_stride;
    double* dkj = dk + j * d_qk;
    double* dvj = dv + j * d_v;
    for (int32_t d = 0; d < d_qk; ++d) dkj[d] = 0.0;
    for (int32_t d = 0; d < d_v; ++d) dvj[d] = 0.0;
    for (int64_t r = 0; r < R; ++r) {
      if (!allowed(pos[r], j, s, l, b, sparse, causal)) continue;
      const float* qr = q + r * q_stride;
      const float* dor = dout + r * do_stride;
      double acc = 0.0;
      for (int32_t d = 0; d < d_qk; ++d) acc += (double)qr[d] * (double)kj[d];
      const double P = exp(scale * acc - m[r]) / L[r];
      double dp = 0.0;
      for (int32_t d = 0; d < d_v; ++d) dp += (double)dor[d] * (double)vj[d];
      const double dz = P * (dp - D[r]);
      for (int32_t d = 0; d < d_qk; ++d) dkj[d] += scale * dz * (double)qr[d];
      for (int32_t d = 0; d < d_v; ++d) dvj[d] += P * (double)dor[d];
    }
  }
  free(m);
  free(L);
  free(D);
}

int loza_oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
