/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU reference for the ParamSpMM hot path
 * (arXiv 2605.15695, /root/reference/PAPER.md; "P:NN" = PAPER.md line NN,
 * "S:NN" = SPEC.md line NN).  It shares no code, header, table or constant
 * with the CUDA library under paper_2605_15695_b200/csrc/ and neither side
 * includes or links the other.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's
 * shared object.  The product path never routes through here.
 *
 * Every function below follows the paper's definition or procedure step by
 * step, in the paper's order and notation, with no blocking, fusion or
 * reordering beyond what that definition states.  Readings of places where
 * the paper is silent or garbled are the ones listed in DESIGN.md §3
 * (SURVEY.md §8(c) c-1a ... c-27).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"):
 *   oracle_spmm_rows     : hand case S:68, identity / permutation / diagonal
 *                          closed forms, dense fp64 brute force (numpy matmul),
 *                          integer-valued exactness, permuted-graph identity.
 *   oracle_gap           : every cell of Table 2.
 *   oracle_pcsr_build    : S:125 worked example, hand-derived pin X,
 *                          V=1 == CSR, lossless scatter-back,
 *                          conservation, bound, c-18.
 *   oracle_pcsr metrics  : PR examples, SG,
 *                          SR.
 *   oracle_features      : 4x4 identity, empty-row case,
 *                          pin X, brute-force numpy statistics, permutation
 *                          invariance.
 * Every function here is pinned.  The config decider has no oracle at all
 * ("parity unpinned", c-4): any valid config is correct if C is.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_ERR_INVALID 1
#define ORACLE_ERR_EMPTY 5
#define ORACLE_ERR_OOM 8

/* ------------------------------------------------------------------------ */
/* c-1  SpMM definition: C = A.B with A n x n sparse (CSR), B n x K dense.   */
/* P:48 "SpMM is defined as A_{n x n} B_{n x dim} = C_{n x dim}";            */
/* P:54 a MAC multiplies a nonzero of A with an element of B and             */
/* accumulates into C; Alg. 1 traverses row i over                 */
/* [rowPtr[i], rowPtr[i+1]).  Accumulation is in fp64 (c-15).         */
/* mag[i,k] = sum_p |a_ip| |b_{col(p),k}| is the scale used by the tolerance */
/* |C_gpu - C| <= 1e-5 mag + 1e-6 stated in BASELINE.json north_star.        */
/*                                                                          */
/* rows == NULL computes all n rows (out row r = matrix row r); otherwise   */
/* out row r = matrix row rows[r].  out / mag have leading dimension K.     */
/* ------------------------------------------------------------------------ */
int oracle_spmm_rows(int64_t n, const int32_t *rowPtr, const int32_t *colIdx,
                     const float *val, const float *B, int64_t ldb, int32_t K,
                     int64_t nrows, const int64_t *rows, double *out,
                     double *mag, int32_t num_threads) {
  if (n < 0 || K < 1 || ldb < K) return ORACLE_ERR_INVALID;
  int64_t count = rows ? nrows : n;
#ifdef _OPENMP
  if (num_threads < 1) num_threads = 1;
#pragma omp parallel for schedule(dynamic, 64) num_threads(num_threads)
#endif
  for (int64_t r = 0; r < count; ++r) {
    int64_t i = rows ? rows[r] : r; /* Crow */
    double *acc = out + r * (int64_t)K;
    double *m = mag ? mag + r * (int64_t)K : NULL;
    for (int32_t k = 0; k < K; ++k) {
      acc[k] = 0.0;
      if (m) m[k] = 0.0;
    }
    if (i < 0 || i >= n) continue;
    int32_t head = rowPtr[i], tail = rowPtr[i + 1];
    for (int32_t p = head; p < tail; ++p) {
      int64_t Brow = colIdx[p];
      double a = (double)val[p];
      const float *b = B + Brow * ldb;
      for (int32_t k = 0; k < K; ++k) {
        acc[k] += a * (double)b[k]; /* one MAC job (Alg.1 l.11) */
        if (m) m[k] += fabs(a) * fabs((double)b[k]);
      }
    }
  }
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* Eq. 1 MAC-job gap with reading c-1a: when            */
/* dim mod (F.omega) == 0 there is no residual warp and the gap is 0, which */
/* is what every cell of Table 2 prints.                        */
/* ------------------------------------------------------------------------ */
int64_t oracle_gap(int64_t dim, int64_t F, int64_t omega) {
  int64_t Fw = F * omega;
  int64_t tn = dim < Fw ? dim : Fw; /* tn = min(dim, F.omega) */
  int64_t tr = dim % Fw;            /* tr = dim mod (F.omega) */
  if (tr == 0) return 0;            /* c-1a */
  return tn - tr;                   /* gap = tn - tr */
}

/* ------------------------------------------------------------------------ */
/* c-2  PCSR generation (P:208 data representation, P:211 generation).     */
/*                                                                          */
/* Step 1  P = ceil(n/V) row panels; panel p covers rows [pV, min(n,pV+V)). */
/* Step 2  vectorized blocking: in each panel the ascending union of its    */
/*         rows' column indices; one V x 1 nonzero vector per column c,     */
/*         val[i*V + k] = A[pV+k, c] or +0.0f where row pV+k lacks c or     */
/*         does not exist ("zero padding", P:228-229 val       */
/*         layout, c-6, c-7, c-8).                                          */
/* Step 3  rowPtr_panel[p+1] = rowPtr_panel[p] + |union_p|.                 */
/* Step 4  S = 0: (rowPtr_panel, colIdx, val), TRow empty.          */
/* Step 5  S = 1: SG = CEILDIV(d^_V, omega) * omega with                    */
/*         d^_V = nnz_V / #non-empty panels (Eq. 3, c-2a, c-3a:  */
/*         integer form ceil(nnz_V / (P^ omega)) omega) or sg_override if   */
/*         nonzero (c-18).  Each panel's run of L vectors becomes           */
/*         max(1, ceil(L/SG)) chunks at offsets 0, SG, 2SG, ... (c-5), rowPtr */
/*         is reassigned to chunk delimiters and TRow[c] = source panel     */
/*         ("rowPtr is reassigned ... TRow is generated").            */
/* Metrics  PR_V = 1 - nnz/(nnz_V V) (Eq. 2);                        */
/*         SR = len(reassigned rowPtr)/len(original rowPtr)                 */
/*            = (chunks+1)/(P+1) (Eq. 4, c-4a).                      */
/* All outputs are malloc'd here and released with oracle_pcsr_free.        */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t n, V, S, omega;
  int64_t num_panels;     /* P */
  int64_t nnz;            /* nonzeros of A */
  int64_t nnz_v;          /* nonzero vectors */
  int64_t nonempty_panels;/* P^ */
  int64_t sg;             /* split granularity used (0 when S = 0) */
  int64_t num_chunks;     /* S = 1: chunks; S = 0: panels */
  int64_t rowptr_len;     /* P+1 (S=0) or chunks+1 (S=1) */
  double pr, sr;
  int32_t *rowPtr, *colIdx, *TRow; /* TRow NULL when S = 0 */
  float *val;
} oracle_pcsr;

void oracle_pcsr_free(oracle_pcsr *p) {
  if (!p) return;
  free(p->rowPtr);
  free(p->colIdx);
  free(p->TRow);
  free(p->val);
  p->rowPtr = p->colIdx = p->TRow = NULL;
  p->val = NULL;
}

/* Smallest column among the heads of the panel's V rows, or -1 if all done. */
static int64_t panel_min_head(int64_t V, const int32_t *colIdx,
                              const int64_t *pos, const int64_t *end) {
  int64_t best = -1;
  for (int64_t k = 0; k < V; ++k)
    if (pos[k] < end[k] && (best < 0 || colIdx[pos[k]] < best))
      best = colIdx[pos[k]];
  return best;
}

int oracle_pcsr_build(int64_t n, const int32_t *rowPtr, const int32_t *colIdx,
                      const float *val, int64_t V, int64_t S, int64_t omega,
                      int64_t sg_override, oracle_pcsr *out) {
  memset(out, 0, sizeof(*out));
  if (n < 1 || V < 1 || V > 64 || (S != 0 && S != 1) || omega < 1 ||
      sg_override < 0)
    return ORACLE_ERR_INVALID;
  out->n = n;
  out->V = V;
  out->S = S;
  out->omega = omega;
  out->nnz = rowPtr[n];

  /* Step 1 */
  int64_t P = (n + V - 1) / V;
  out->num_panels = P;

  int64_t pos[64], end[64];
  /* Steps 2-3, first pass: |union_p| for every panel. */
  int32_t *panelPtr = (int32_t *)malloc((size_t)(P + 1) * sizeof(int32_t));
  if (!panelPtr) return ORACLE_ERR_OOM;
  panelPtr[0] = 0;
  int64_t total = 0;
  for (int64_t p = 0; p < P; ++p) {
    for (int64_t k = 0; k < V; ++k) {
      int64_t r = p * V + k;
      pos[k] = r < n ? rowPtr[r] : 0;
      end[k] = r < n ? rowPtr[r + 1] : 0;
    }
    int64_t L = 0;
    for (;;) {
      int64_t c = panel_min_head(V, colIdx, pos, end);
      if (c < 0) break;
      for (int64_t k = 0; k < V; ++k)
        if (pos[k] < end[k] && colIdx[pos[k]] == c) pos[k]++;
      L++;
    }
    total += L;
    if (total > INT32_MAX) {
      free(panelPtr);
      return ORACLE_ERR_INVALID;
    }
    panelPtr[p + 1] = (int32_t)total;
  }
  int64_t nnz_v = total;
  out->nnz_v = nnz_v;

  /* Step 2, second pass: colIdx and the V values of every vector. */
  int32_t *vcol = (int32_t *)malloc((size_t)(nnz_v > 0 ? nnz_v : 1) * sizeof(int32_t));
  float *vval = (float *)malloc((size_t)(nnz_v > 0 ? nnz_v * V : 1) * sizeof(float));
  if (!vcol || !vval) {
    free(panelPtr); free(vcol); free(vval);
    return ORACLE_ERR_OOM;
  }
  for (int64_t p = 0; p < P; ++p) {
    for (int64_t k = 0; k < V; ++k) {
      int64_t r = p * V + k;
      pos[k] = r < n ? rowPtr[r] : 0;
      end[k] = r < n ? rowPtr[r + 1] : 0;
    }
    int64_t i = panelPtr[p];
    for (;;) {
      int64_t c = panel_min_head(V, colIdx, pos, end);
      if (c < 0) break;
      vcol[i] = (int32_t)c;
      for (int64_t k = 0; k < V; ++k) {
        if (pos[k] < end[k] && colIdx[pos[k]] == c) {
          vval[i * V + k] = val[pos[k]];
          pos[k]++;
        } else {
          vval[i * V + k] = 0.0f; /* zero padding, +0.0f (c-7) */
        }
      }
      i++;
    }
  }
  out->colIdx = vcol;
  out->val = vval;

  int64_t nonempty = 0;
  for (int64_t p = 0; p < P; ++p)
    if (panelPtr[p + 1] > panelPtr[p]) nonempty++;
  out->nonempty_panels = nonempty;

  /* Eq. 2 */
  out->pr = nnz_v > 0 ? 1.0 - (double)out->nnz / ((double)nnz_v * (double)V)
                      : NAN;

  if (S == 0) {
    /* Step 4 */
    out->rowPtr = panelPtr;
    out->TRow = NULL;
    out->sg = 0;
    out->num_chunks = P;
    out->rowptr_len = P + 1;
    out->sr = 1.0;
    return ORACLE_OK;
  }

  /* Step 5: SG (Eq. 3) */
  int64_t SG;
  if (sg_override > 0) {
    SG = sg_override;
  } else {
    if (nonempty == 0) { /* SG undefined on an all-empty matrix */
      free(panelPtr);
      oracle_pcsr_free(out);
      return ORACLE_ERR_EMPTY;
    }
    int64_t denom = nonempty * omega;
    SG = ((nnz_v + denom - 1) / denom) * omega; /* ceil(d^_V/omega)*omega */
  }
  out->sg = SG;

  int64_t chunks = 0;
  for (int64_t p = 0; p < P; ++p) {
    int64_t L = panelPtr[p + 1] - panelPtr[p];
    chunks += L == 0 ? 1 : (L + SG - 1) / SG; /* max(1, ceil(L/SG)), c-5 */
  }
  int32_t *chunkPtr = (int32_t *)malloc((size_t)(chunks + 1) * sizeof(int32_t));
  int32_t *trow = (int32_t *)malloc((size_t)chunks * sizeof(int32_t));
  if (!chunkPtr || !trow) {
    free(panelPtr); free(chunkPtr); free(trow);
    oracle_pcsr_free(out);
    return ORACLE_ERR_OOM;
  }
  int64_t c = 0;
  for (int64_t p = 0; p < P; ++p) {
    int64_t L = panelPtr[p + 1] - panelPtr[p];
    int64_t nch = L == 0 ? 1 : (L + SG - 1) / SG;
    for (int64_t j = 0; j < nch; ++j) {
      chunkPtr[c] = (int32_t)(panelPtr[p] + j * SG);
      trow[c] = (int32_t)p;
      c++;
    }
  }
  chunkPtr[chunks] = (int32_t)nnz_v;
  free(panelPtr);
  out->rowPtr = chunkPtr;
  out->TRow = trow;
  out->num_chunks = chunks;
  out->rowptr_len = chunks + 1;
  out->sr = (double)(chunks + 1) / (double)(P + 1); /* Eq. 4 */
  return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* c-3  Table 3 features with readings c-19..c-22 (S:271-278,   */
/* S:289-290).  Order of the 16 outputs:                                    */
/*  0 n, 1 n_hat, 2 nnz, 3 delta, 4 d, 5 d_hat, 6 d_max, 7 cv, 8 cv_hat,    */
/*  9 sr1, 10 sr2, 11 rho, 12 b, 13 b_max, 14 pr1, 15 pr2                    */
/* ------------------------------------------------------------------------ */
int oracle_features(int64_t n, const int32_t *rowPtr, const int32_t *colIdx,
                    const float *val, int64_t omega, double *f) {
  if (n < 1 || omega < 1) return ORACLE_ERR_INVALID;
  int64_t nnz = rowPtr[n];
  if (nnz == 0) return ORACLE_ERR_EMPTY;

  int64_t n_hat = 0, d_max = 0, b_max = 0;
  double b_sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t deg = rowPtr[i + 1] - rowPtr[i]; /* out-degree, c-22 */
    if (deg > 0) n_hat++;
    if (deg > d_max) d_max = deg;
    /* row bandwidth: last col - first col (P:329 footnote); empty -> 0 (c-21) */
    int64_t bw = deg > 0 ? (int64_t)colIdx[rowPtr[i + 1] - 1] - colIdx[rowPtr[i]] : 0;
    if (bw > b_max) b_max = bw;
    b_sum += (double)bw;
  }
  double d = (double)nnz / (double)n;
  double d_hat = (double)nnz / (double)n_hat;
  /* CV = population std / mean over all n rows; CV^ over non-empty rows (c-20) */
  double ss = 0.0, ss_hat = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double deg = (double)(rowPtr[i + 1] - rowPtr[i]);
    ss += (deg - d) * (deg - d);
    if (deg > 0) ss_hat += (deg - d_hat) * (deg - d_hat);
  }
  double cv = sqrt(ss / (double)n) / d;
  double cv_hat = sqrt(ss_hat / (double)n_hat) / d_hat;

  /* SR_i under <V=i, S=true> and PR_i under V=i, via the PCSR procedure. */
  oracle_pcsr p1, p2;
  int st = oracle_pcsr_build(n, rowPtr, colIdx, val, 1, 1, omega, 0, &p1);
  if (st) return st;
  st = oracle_pcsr_build(n, rowPtr, colIdx, val, 2, 1, omega, 0, &p2);
  if (st) {
    oracle_pcsr_free(&p1);
    return st;
  }
  f[0] = (double)n;
  f[1] = (double)n_hat;
  f[2] = (double)nnz;
  f[3] = (double)n_hat / (double)n;
  f[4] = d;
  f[5] = d_hat;
  f[6] = (double)d_max;
  f[7] = cv;
  f[8] = cv_hat;
  f[9] = p1.sr;
  f[10] = p2.sr;
  f[11] = (double)nnz / ((double)n * (double)n);
  f[12] = b_sum / (double)n;
  f[13] = (double)b_max;
  f[14] = p1.pr;
  f[15] = p2.pr;
  oracle_pcsr_free(&p1);
  oracle_pcsr_free(&p2);
  return ORACLE_OK;
}
