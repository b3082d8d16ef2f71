/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the FastTuckerPlus hot path.
 *
 * A plain-C restatement of the reference's fp32 FastTuckerPlus epoch
 * (/root/reference/proj/src/decomposition.cpp:623-705) and its fp64
 * evaluation (evaluation.cpp:36-72, model.cpp:70-92), written from the
 * algorithm, not copied.  It reproduces the reference's exact rounding
 * sequence: IEEE fp32 multiply then add, no FMA
 * contraction (built with -ffp-contract=off and no -march, like the
 * reference's own Release build), summations in the reference's index order
 * over 16-padded tile extents, padding cells exactly +0.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function here
 * bit-for-bit against the reference library itself (oracle/_ref, built from
 * /root/reference by oracle/Makefile) and against the committed golden
 * fixtures in tests/golden/ (generated from oracle/_ref by
 * oracle/gen_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * call into this file.  The B200 engine never links it.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FO_TILE 16
#define FO_MAXN 8

static int pad16(int x) { return (x + FO_TILE - 1) / FO_TILE * FO_TILE; }

/* Padded per-batch workspace, all dense row-major with 16-padded extents. */
typedef struct {
  int order, cap, capp, r, rp;
  int j[FO_MAXN], jp[FO_MAXN];
  float *a[FO_MAXN]; /* capp x jp   staged factor rows (decomposition.cpp:170-184) */
  float *c[FO_MAXN]; /* capp x rp   C = A_psi B (decomposition.cpp:186-196)      */
  float *d[FO_MAXN]; /* capp x rp   D = hadamard of the other C (:200-212)       */
  float *u[FO_MAXN]; /* capp x jp   U = D B^T (:226-232)                          */
  float *bp[FO_MAXN];  /* jp x rp  padded B snapshot (CoreTiles, :57-72)        */
  float *btp[FO_MAXN]; /* rp x jp  padded B^T                                    */
  float *xhat, *resid; /* cap */
} fo_ws;

static void ws_free(fo_ws* w) {
  for (int n = 0; n < w->order; ++n) {
    free(w->a[n]); free(w->c[n]); free(w->d[n]); free(w->u[n]);
    free(w->bp[n]); free(w->btp[n]);
  }
  free(w->xhat); free(w->resid);
}

static int ws_init(fo_ws* w, int order, const int32_t* ranks, int r, int cap) {
  memset(w, 0, sizeof *w);
  if (order < 1 || order > FO_MAXN) return 1;
  w->order = order; w->cap = cap; w->capp = pad16(cap);
  w->r = r; w->rp = pad16(r);
  for (int n = 0; n < order; ++n) {
    w->j[n] = ranks[n]; w->jp[n] = pad16(ranks[n]);
    w->a[n] = calloc((size_t)w->capp * w->jp[n], sizeof(float));
    w->c[n] = calloc((size_t)w->capp * w->rp, sizeof(float));
    w->d[n] = calloc((size_t)w->capp * w->rp, sizeof(float));
    w->u[n] = calloc((size_t)w->capp * w->jp[n], sizeof(float));
    w->bp[n] = calloc((size_t)w->jp[n] * w->rp, sizeof(float));
    w->btp[n] = calloc((size_t)w->rp * w->jp[n], sizeof(float));
  }
  w->xhat = calloc((size_t)cap, sizeof(float));
  w->resid = calloc((size_t)cap, sizeof(float));
  return 0;
}

/* CoreTiles snapshot: zero-padded B and B^T (decomposition.cpp:57-72). */
static void ws_snapshot_b(fo_ws* w, float* const* b) {
  for (int n = 0; n < w->order; ++n) {
    memset(w->bp[n], 0, sizeof(float) * w->jp[n] * w->rp);
    memset(w->btp[n], 0, sizeof(float) * w->rp * w->jp[n]);
    for (int j = 0; j < w->j[n]; ++j)
      for (int c = 0; c < w->r; ++c) {
        float v = b[n][(size_t)j * w->r + c];
        w->bp[n][j * w->rp + c] = v;
        w->btp[n][c * w->jp[n] + j] = v;
      }
  }
}

/* Dense padded product out = x (rows x k) * y (k x cols), accumulation
 * starting from +0 in ascending k over the padded inner extent: the
 * tile_mma / matmul_tiled order (tiles.cpp:21-47), no FMA. */
static void mm(const float* x, const float* y, float* out, int rows, int k,
               int cols) {
  for (int i = 0; i < rows; ++i)
    for (int c = 0; c < cols; ++c) {
      float acc = 0.0f;
      for (int q = 0; q < k; ++q) {
        float p = x[i * k + q] * y[q * cols + c];
        acc = acc + p;
      }
      out[i * cols + c] = acc;
    }
}

/* Stages factor rows and computes C and D for one batch (decomposition.cpp
 * :170-212).  idx is [order][cap] (padding rows index 0), a_src the model's
 * factor matrices. */
static void fo_stage_cd(fo_ws* w, float* const* amat, const int32_t* idx,
                        int m_eff) {
  const int order = w->order;
  for (int n = 0; n < order; ++n) {
    memset(w->a[n], 0, sizeof(float) * w->capp * w->jp[n]);
    for (int m = 0; m < m_eff; ++m) {
      const float* row = amat[n] + (size_t)idx[n * w->cap + m] * w->j[n];
      for (int j = 0; j < w->j[n]; ++j) w->a[n][m * w->jp[n] + j] = row[j];
    }
    mm(w->a[n], w->bp[n], w->c[n], w->capp, w->jp[n], w->rp);
  }
  /* D^(k) = C^(first) copied, then multiplied by C^(n) for n > first,
   * n != k, modes ascending (decomposition.cpp:203-210). */
  for (int k = 0; k < order; ++k) {
    int first = (k == 0) ? 1 : 0;
    if (order == 1) first = 0;
    memcpy(w->d[k], w->c[first], sizeof(float) * w->capp * w->rp);
    for (int n = first + 1; n < order; ++n) {
      if (n == k) continue;
      for (int i = 0; i < w->capp * w->rp; ++i) w->d[k][i] = w->d[k][i] * w->c[n][i];
    }
  }
}

/* Storage scheme (store_c): C rows taken from the C cache instead of the
 * tile product.  A cache row is CCache::refresh's sum over the unpadded J,
 * j ascending, multiply then add (decomposition.cpp:89-107), copied in for
 * m < m_eff and zero below (stage_c_rows_from_cache, :299-314); computing the
 * touched rows on the fly gives the same values as building the whole cache. */
static void fo_stage_cd_cached(fo_ws* w, float* const* amat, float* const* bmat,
                               const int32_t* idx, int m_eff) {
  const int order = w->order;
  for (int n = 0; n < order; ++n) {
    memset(w->a[n], 0, sizeof(float) * w->capp * w->jp[n]);
    memset(w->c[n], 0, sizeof(float) * w->capp * w->rp);
    for (int m = 0; m < m_eff; ++m) {
      const float* row = amat[n] + (size_t)idx[n * w->cap + m] * w->j[n];
      for (int j = 0; j < w->j[n]; ++j) w->a[n][m * w->jp[n] + j] = row[j];
      for (int c = 0; c < w->r; ++c) {
        float acc = 0.0f;
        for (int j = 0; j < w->j[n]; ++j) {
          float p = row[j] * bmat[n][(size_t)j * w->r + c];
          acc = acc + p;
        }
        w->c[n][m * w->rp + c] = acc;
      }
    }
  }
  for (int k = 0; k < order; ++k) {
    int first = (k == 0) ? 1 : 0;
    if (order == 1) first = 0;
    memcpy(w->d[k], w->c[first], sizeof(float) * w->capp * w->rp);
    for (int n = first + 1; n < order; ++n) {
      if (n == k) continue;
      for (int i = 0; i < w->capp * w->rp; ++i) w->d[k][i] = w->d[k][i] * w->c[n][i];
    }
  }
}

/* U^(n) = D^(n) B^(n)T (decomposition.cpp:226-232). */
static void fo_u(fo_ws* w) {
  for (int n = 0; n < w->order; ++n)
    mm(w->d[n], w->btp[n], w->u[n], w->capp, w->rp, w->jp[n]);
}

/* row_dot over the padded extent (tiles.cpp:86-99) then the residual rule
 * (decomposition.cpp:234-238). */
static void fo_predict_rows(fo_ws* w, const float* x, const float* p,
                            const float* q, int ld, int m_eff) {
  for (int m = 0; m < w->cap; ++m) {
    float acc = 0.0f;
    for (int k = 0; k < ld; ++k) {
      float t = p[m * ld + k] * q[m * ld + k];
      acc = acc + t;
    }
    w->xhat[m] = acc;
    w->resid[m] = (m < m_eff) ? x[m] - acc : 0.0f;
  }
}

/* Factor-side prediction: A^(1)_psi against U^(1) (decomposition.cpp:240-245). */
static void fo_predict_factor_side(fo_ws* w, const float* x, int m_eff) {
  fo_predict_rows(w, x, w->a[0], w->u[0], w->jp[0], m_eff);
}

/* C-side prediction: C^(1) against D^(1) (decomposition.cpp:247-252). */
static void fo_predict_c_side(fo_ws* w, const float* x, int m_eff) {
  fo_predict_rows(w, x, w->c[0], w->d[0], w->rp, m_eff);
}

/* Eq. (14) simultaneous factor update from the staged snapshot, modes then
 * rows ascending, later duplicate rows win (decomposition.cpp:254-275). */
static void fo_update_factors(fo_ws* w, float* const* amat, const int32_t* idx,
                              int m_eff, float lr_a, float reg_a) {
  for (int n = 0; n < w->order; ++n)
    for (int m = 0; m < m_eff; ++m) {
      const float rm = w->resid[m];
      float* dst = amat[n] + (size_t)idx[n * w->cap + m] * w->j[n];
      for (int j = 0; j < w->j[n]; ++j) {
        float snap = w->a[n][m * w->jp[n] + j];
        float uu = w->u[n][m * w->jp[n] + j];
        float g = rm * uu;
        float rg = reg_a * snap;
        float step = lr_a * (g - rg);
        dst[j] = snap + step;
      }
    }
}

/* Eq. (15) per-batch core gradient E^T D with E = resid (x) A_psi, summed
 * over padded batch rows ascending, added into acc (decomposition.cpp
 * :277-296). */
static void fo_core_grads(fo_ws* w, float* const* acc) {
  for (int n = 0; n < w->order; ++n)
    for (int j = 0; j < w->j[n]; ++j)
      for (int c = 0; c < w->r; ++c) {
        float g = 0.0f;
        for (int m = 0; m < w->capp; ++m) {
          float rm = (m < w->cap) ? w->resid[m] : 0.0f;
          float e = rm * w->a[n][m * w->jp[n] + j];
          float p = e * w->d[n][m * w->rp + c];
          g = g + p;
        }
        float* dst = acc[n] + (size_t)j * w->r + c;
        *dst = *dst + g;
      }
}

static void gather_batch(int order, const int32_t* idx_aos, const float* vals,
                         const int64_t* pos, int m_eff, int cap, int32_t* idx,
                         float* x) {
  for (int m = 0; m < cap; ++m) {
    x[m] = 0.0f;
    for (int n = 0; n < order; ++n) idx[n * cap + m] = 0;
  }
  for (int m = 0; m < m_eff; ++m) {
    int64_t p = pos[m];
    x[m] = vals[p];
    for (int n = 0; n < order; ++n) idx[n * cap + m] = idx_aos[p * order + n];
  }
}

/* ------------------------------------------------------------------------ */
/* Public entry points (ctypes).                                            */

/* One batch through the per-batch pipeline; same output layout as
 * oracle/ref_capi.cpp:ref_batch_probe.  Mutates amat like
 * update_factors_plus. */
int fo_batch_probe(int order, const int32_t* ranks, int r, float* const* amat,
                   float* const* bmat, const int32_t* idx_aos,
                   const float* vals, const int64_t* rows, int m_eff, int cap,
                   float lr_a, float reg_a, float* c_out, float* d_out,
                   float* u_out, float* xhat_f, float* resid_f, float* xhat_c,
                   float* resid_c, float* a_new, float* g_out) {
  fo_ws w;
  if (ws_init(&w, order, ranks, r, cap)) return 1;
  int jmax = 0;
  for (int n = 0; n < order; ++n) jmax = ranks[n] > jmax ? ranks[n] : jmax;
  int32_t* idx = malloc(sizeof(int32_t) * order * cap);
  float* x = malloc(sizeof(float) * cap);
  gather_batch(order, idx_aos, vals, rows, m_eff, cap, idx, x);
  ws_snapshot_b(&w, bmat);
  fo_stage_cd(&w, amat, idx, m_eff);
  fo_u(&w);
  fo_predict_factor_side(&w, x, m_eff);
  for (int n = 0; n < order; ++n)
    for (int m = 0; m < cap; ++m) {
      for (int c = 0; c < r; ++c) {
        c_out[((size_t)n * cap + m) * r + c] = w.c[n][m * w.rp + c];
        d_out[((size_t)n * cap + m) * r + c] = w.d[n][m * w.rp + c];
      }
      for (int j = 0; j < ranks[n]; ++j)
        u_out[((size_t)n * cap + m) * jmax + j] = w.u[n][m * w.jp[n] + j];
    }
  memcpy(xhat_f, w.xhat, sizeof(float) * cap);
  memcpy(resid_f, w.resid, sizeof(float) * cap);
  fo_update_factors(&w, amat, idx, m_eff, lr_a, reg_a);
  for (int n = 0; n < order; ++n)
    for (int m = 0; m < m_eff; ++m)
      for (int j = 0; j < ranks[n]; ++j)
        a_new[((size_t)n * cap + m) * jmax + j] =
            amat[n][(size_t)idx[n * cap + m] * ranks[n] + j];
  fo_predict_c_side(&w, x, m_eff);
  memcpy(xhat_c, w.xhat, sizeof(float) * cap);
  memcpy(resid_c, w.resid, sizeof(float) * cap);
  float* acc[FO_MAXN];
  for (int n = 0; n < order; ++n) acc[n] = calloc((size_t)ranks[n] * r, sizeof(float));
  fo_core_grads(&w, acc);
  for (int n = 0; n < order; ++n) {
    for (int j = 0; j < ranks[n]; ++j)
      for (int c = 0; c < r; ++c)
        g_out[((size_t)n * jmax + j) * r + c] = acc[n][(size_t)j * r + c];
    free(acc[n]);
  }
  free(idx); free(x);
  ws_free(&w);
  return 0;
}

/* Factor phase (HOT LOOP 1) with workers = 1: batches of `cap` positions of
 * perm in order, each seeing all earlier writes (decomposition.cpp:637-661). */
int fo_factor_phase(int order, const int32_t* ranks, int r, float* const* amat,
                    float* const* bmat, int64_t nnz, const int32_t* idx_aos,
                    const float* vals, const int64_t* perm, int cap,
                    float lr_a, float reg_a) {
  fo_ws w;
  if (ws_init(&w, order, ranks, r, cap)) return 1;
  int32_t* idx = malloc(sizeof(int32_t) * order * cap);
  float* x = malloc(sizeof(float) * cap);
  ws_snapshot_b(&w, bmat);
  for (int64_t off = 0; off < nnz; off += cap) {
    int m_eff = (int)((nnz - off) < cap ? (nnz - off) : cap);
    gather_batch(order, idx_aos, vals, perm + off, m_eff, cap, idx, x);
    fo_stage_cd(&w, amat, idx, m_eff);
    fo_u(&w);
    fo_predict_factor_side(&w, x, m_eff);
    fo_update_factors(&w, amat, idx, m_eff, lr_a, reg_a);
  }
  free(idx); free(x);
  ws_free(&w);
  return 0;
}

/* Core phase (HOT LOOP 2) with workers = 1: per-batch E^T D accumulated in
 * batch order, merged into a zero total, applied once (decomposition.cpp
 * :663-703, :146-162, :576-589).  grad_out (optional) receives the merged
 * total, [order][J_n*R] concatenated. */
int fo_core_phase(int order, const int32_t* ranks, int r, float* const* amat,
                  float* const* bmat, int64_t nnz, const int32_t* idx_aos,
                  const float* vals, const int64_t* perm, int cap, float lr_b,
                  float reg_b, float* grad_out, int store_c) {
  if (nnz <= 0) return 2; /* apply_core_update: empty tensor */
  fo_ws w;
  if (ws_init(&w, order, ranks, r, cap)) return 1;
  int32_t* idx = malloc(sizeof(int32_t) * order * cap);
  float* x = malloc(sizeof(float) * cap);
  float* acc[FO_MAXN];
  for (int n = 0; n < order; ++n) acc[n] = calloc((size_t)ranks[n] * r, sizeof(float));
  ws_snapshot_b(&w, bmat);
  for (int64_t off = 0; off < nnz; off += cap) {
    int m_eff = (int)((nnz - off) < cap ? (nnz - off) : cap);
    gather_batch(order, idx_aos, vals, perm + off, m_eff, cap, idx, x);
    if (store_c) fo_stage_cd_cached(&w, amat, bmat, idx, m_eff);
    else fo_stage_cd(&w, amat, idx, m_eff);
    fo_predict_c_side(&w, x, m_eff);
    fo_core_grads(&w, acc);
  }
  const float inv = 1.0f / (float)nnz;
  size_t off = 0;
  for (int n = 0; n < order; ++n) {
    size_t len = (size_t)ranks[n] * r;
    for (size_t i = 0; i < len; ++i) {
      float total = 0.0f + acc[n][i]; /* CoreGradAccumulator::merge into zero */
      if (grad_out) grad_out[off + i] = total;
      float b = bmat[n][i];
      float gi = total * inv;
      float rb = reg_b * b;
      float step = lr_b * (gi - rb);
      bmat[n][i] = b + step;
    }
    off += len;
    free(acc[n]);
  }
  free(idx); free(x);
  ws_free(&w);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* FastTucker baseline (decomposition.cpp:707-770), workers = 1.            */

/* Rows of every mode except `skip` staged (zero padding), C = A_psi B from
 * the padded snapshot (stage_factor_rows_impl / compute_c_batch_impl with a
 * skip mode, decomposition.cpp:170-196), and D of `mode` alone
 * (compute_d_single_impl, :214-224). */
static void ft_stage_cd(fo_ws* w, float* const* amat, const int32_t* idx, int m_eff,
                        int skip, int mode) {
  for (int n = 0; n < w->order; ++n) {
    memset(w->a[n], 0, sizeof(float) * w->capp * w->jp[n]);
    for (int m = 0; m < m_eff; ++m) {
      const float* row = amat[n] + (size_t)idx[n * w->cap + m] * w->j[n];
      for (int j = 0; j < w->j[n]; ++j) w->a[n][m * w->jp[n] + j] = row[j];
    }
    if (n == mode && skip == mode) continue;
    if (n != mode) mm(w->a[n], w->bp[n], w->c[n], w->capp, w->jp[n], w->rp);
  }
  int first = (mode == 0) ? 1 : 0;
  memcpy(w->d[mode], w->c[first], sizeof(float) * w->capp * w->rp);
  for (int n = first + 1; n < w->order; ++n) {
    if (n == mode) continue;
    for (int i = 0; i < w->capp * w->rp; ++i) w->d[mode][i] = w->d[mode][i] * w->c[n][i];
  }
}

/* Factor block of `mode` over a per-bucket plan: bucket b's entries are
 * perm[boff[b] .. boff[b+1]), cut into batches of cap; each batch moves the
 * bucket's shared row by the 1/M-mean gradient (update_factor_fasttucker_impl,
 * :316-371). */
int fo_fasttucker_factor_block(int order, const int32_t* ranks, int r, float* const* amat,
                               float* const* bmat, const int32_t* idx_aos, const float* vals,
                               const int64_t* perm, const int64_t* boff, int64_t nb, int cap,
                               int mode, float lr_a, float reg_a) {
  fo_ws w;
  if (order < 2 || ws_init(&w, order, ranks, r, cap)) return 1;
  int32_t* idx = malloc(sizeof(int32_t) * order * cap);
  float* x = malloc(sizeof(float) * cap);
  const int jn = ranks[mode];
  float* snap = malloc(sizeof(float) * jn);
  float* cs = malloc(sizeof(float) * r);
  ws_snapshot_b(&w, bmat);
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t off = boff[b]; off < boff[b + 1]; off += cap) {
      int m_eff = (int)((boff[b + 1] - off) < cap ? (boff[b + 1] - off) : cap);
      gather_batch(order, idx_aos, vals, perm + off, m_eff, cap, idx, x);
      const int32_t row = idx[mode * cap];
      ft_stage_cd(&w, amat, idx, m_eff, mode, mode);
      mm(w.d[mode], w.btp[mode], w.u[mode], w.capp, w.rp, w.jp[mode]);
      float* dst = amat[mode] + (size_t)row * jn;
      for (int j = 0; j < jn; ++j) snap[j] = dst[j];
      for (int c = 0; c < r; ++c) { /* c = a B^(n), unpadded j */
        float acc = 0.0f;
        for (int j = 0; j < jn; ++j) {
          float p = snap[j] * bmat[mode][(size_t)j * r + c];
          acc = acc + p;
        }
        cs[c] = acc;
      }
      for (int m = 0; m < m_eff; ++m) { /* x_hat = c . d_m, unpadded R */
        float acc = 0.0f;
        for (int c = 0; c < r; ++c) {
          float p = cs[c] * w.d[mode][m * w.rp + c];
          acc = acc + p;
        }
        w.resid[m] = x[m] - acc;
      }
      const float inv = 1.0f / (float)m_eff;
      for (int j = 0; j < jn; ++j) {
        float g = 0.0f;
        for (int m = 0; m < m_eff; ++m) {
          float p = w.resid[m] * w.u[mode][m * w.jp[mode] + j];
          g = g + p;
        }
        float gi = g * inv;
        float rg = reg_a * snap[j];
        float step = lr_a * (gi - rg);
        dst[j] = snap[j] + step;
      }
    }
  free(idx); free(x); free(snap); free(cs);
  ws_free(&w);
  return 0;
}

/* Core block of `mode` over a global plan: C of the other modes from the
 * block-entry snapshot, C^(n) from the current B^(n), C-side residual,
 * G = (r (x) A_psi)^T D over the padded batch, and B^(n) moves after every
 * batch (update_core_fasttucker_impl, :373-417). */
int fo_fasttucker_core_block(int order, const int32_t* ranks, int r, float* const* amat,
                             float* const* bmat, int64_t nnz, const int32_t* idx_aos,
                             const float* vals, const int64_t* perm, int cap, int mode,
                             float lr_b, float reg_b) {
  fo_ws w;
  if (order < 2 || ws_init(&w, order, ranks, r, cap)) return 1;
  int32_t* idx = malloc(sizeof(int32_t) * order * cap);
  float* x = malloc(sizeof(float) * cap);
  const int jn = ranks[mode];
  ws_snapshot_b(&w, bmat);
  for (int64_t off = 0; off < nnz; off += cap) {
    int m_eff = (int)((nnz - off) < cap ? (nnz - off) : cap);
    gather_batch(order, idx_aos, vals, perm + off, m_eff, cap, idx, x);
    ft_stage_cd(&w, amat, idx, m_eff, -1, mode);
    /* the current B^(n), padded */
    memset(w.bp[mode], 0, sizeof(float) * w.jp[mode] * w.rp);
    for (int j = 0; j < jn; ++j)
      for (int c = 0; c < r; ++c) w.bp[mode][j * w.rp + c] = bmat[mode][(size_t)j * r + c];
    mm(w.a[mode], w.bp[mode], w.c[mode], w.capp, w.jp[mode], w.rp);
    fo_predict_rows(&w, x, w.c[mode], w.d[mode], w.rp, m_eff);
    const float inv = 1.0f / (float)m_eff;
    for (int j = 0; j < jn; ++j)
      for (int c = 0; c < r; ++c) {
        float g = 0.0f;
        for (int m = 0; m < w.capp; ++m) {
          float rm = (m < w.cap) ? w.resid[m] : 0.0f;
          float e = rm * w.a[mode][m * w.jp[mode] + j];
          float p = e * w.d[mode][m * w.rp + c];
          g = g + p;
        }
        float* bb = bmat[mode] + (size_t)j * r + c;
        float gi = g * inv;
        float rb = reg_b * *bb;
        float step = lr_b * (gi - rb);
        *bb = *bb + step;
      }
  }
  free(idx); free(x);
  ws_free(&w);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* FasterTucker baseline (decomposition.cpp:772-843), workers = 1.          */

/* CCache::refresh of one mode (decomposition.cpp:89-107): C_n[i][c] = sum_j
 * A_n[i][j] B_n[j][c], j ascending over the unpadded J. */
void fo_ccache_refresh(int32_t rows, int jn, int r, const float* a, const float* b, float* c) {
  for (int32_t i = 0; i < rows; ++i)
    for (int col = 0; col < r; ++col) {
      float acc = 0.0f;
      for (int j = 0; j < jn; ++j) {
        float p = a[(size_t)i * jn + j] * b[(size_t)j * r + col];
        acc = acc + p;
      }
      c[(size_t)i * r + col] = acc;
    }
}

/* The batch's shared d row: the cached C rows of every other mode, first
 * copied, the rest multiplied in, modes ascending (:420-449). */
static void fst_d_row(int order, int r, int mode, float* const* cmat, const int32_t* e, float* d) {
  int first = 1;
  for (int k = 0; k < order; ++k) {
    if (k == mode) continue;
    const float* crow = cmat[k] + (size_t)e[k] * r;
    for (int c = 0; c < r; ++c) d[c] = first ? crow[c] : d[c] * crow[c];
    first = 0;
  }
}

/* Factor block over a complement-keyed per-bucket plan: batch b is
 * perm[boff[b] .. boff[b+1]); t = B^(n) d, then per-row single-sample steps
 * from the staged rows (update_factor_fastertucker_impl, :451-489); the
 * mode's cache rows are refreshed at the end (:810). */
int fo_fastertucker_factor_block(int order, const int32_t* dims, const int32_t* ranks, int r,
                                 float* const* amat, float* const* bmat, float* const* cmat,
                                 const int32_t* idx_aos, const float* vals, const int64_t* perm,
                                 const int64_t* boff, int64_t nb, int mode, float lr_a,
                                 float reg_a) {
  const int jn = ranks[mode];
  float* d = malloc(sizeof(float) * r);
  float* t = malloc(sizeof(float) * jn);
  int64_t cap = 1;
  for (int64_t b = 0; b < nb; ++b) if (boff[b + 1] - boff[b] > cap) cap = boff[b + 1] - boff[b];
  float* snap = malloc(sizeof(float) * cap * jn);
  float* res = malloc(sizeof(float) * cap);
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t beg = boff[b];
    const int m_eff = (int)(boff[b + 1] - beg);
    fst_d_row(order, r, mode, cmat, idx_aos + (size_t)perm[beg] * order, d);
    for (int m = 0; m < m_eff; ++m) {
      const float* row = amat[mode] + (size_t)idx_aos[(size_t)perm[beg + m] * order + mode] * jn;
      for (int j = 0; j < jn; ++j) snap[m * jn + j] = row[j];
    }
    for (int j = 0; j < jn; ++j) {
      float acc = 0.0f;
      for (int c = 0; c < r; ++c) {
        float p = bmat[mode][(size_t)j * r + c] * d[c];
        acc = acc + p;
      }
      t[j] = acc;
    }
    for (int m = 0; m < m_eff; ++m) {
      float acc = 0.0f;
      for (int j = 0; j < jn; ++j) {
        float p = snap[m * jn + j] * t[j];
        acc = acc + p;
      }
      res[m] = vals[perm[beg + m]] - acc;
    }
    for (int m = 0; m < m_eff; ++m) {
      float* dst = amat[mode] + (size_t)idx_aos[(size_t)perm[beg + m] * order + mode] * jn;
      for (int j = 0; j < jn; ++j) {
        float g = res[m] * t[j];
        float rg = reg_a * snap[m * jn + j];
        float step = lr_a * (g - rg);
        dst[j] = snap[m * jn + j] + step;
      }
    }
  }
  fo_ccache_refresh(dims[mode], jn, r, amat[mode], bmat[mode], cmat[mode]);
  free(d); free(t); free(snap); free(res);
  return 0;
}

/* Core block: residuals from the block-entry cache rows of the mode,
 * g = A_psi^T r, B^(n) += lr (g d^T / M - reg B) after every batch
 * (update_core_fastertucker_impl, :491-533); refresh at the end (:837). */
int fo_fastertucker_core_block(int order, const int32_t* dims, const int32_t* ranks, int r,
                               float* const* amat, float* const* bmat, float* const* cmat,
                               const int32_t* idx_aos, const float* vals, const int64_t* perm,
                               const int64_t* boff, int64_t nb, int mode, float lr_b,
                               float reg_b) {
  const int jn = ranks[mode];
  float* d = malloc(sizeof(float) * r);
  float* g = malloc(sizeof(float) * jn);
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t beg = boff[b];
    const int m_eff = (int)(boff[b + 1] - beg);
    fst_d_row(order, r, mode, cmat, idx_aos + (size_t)perm[beg] * order, d);
    for (int j = 0; j < jn; ++j) g[j] = 0.0f;
    for (int m = 0; m < m_eff; ++m) {
      const int32_t i = idx_aos[(size_t)perm[beg + m] * order + mode];
      const float* crow = cmat[mode] + (size_t)i * r;
      float acc = 0.0f;
      for (int c = 0; c < r; ++c) {
        float p = crow[c] * d[c];
        acc = acc + p;
      }
      const float rm = vals[perm[beg + m]] - acc;
      const float* arow = amat[mode] + (size_t)i * jn;
      for (int j = 0; j < jn; ++j) {
        float p = rm * arow[j];
        g[j] = g[j] + p;
      }
    }
    const float inv = 1.0f / (float)m_eff;
    for (int j = 0; j < jn; ++j)
      for (int c = 0; c < r; ++c) {
        float* bb = bmat[mode] + (size_t)j * r + c;
        float gd = g[j] * d[c];
        float x = gd * inv;
        float rb = reg_b * *bb;
        float step = lr_b * (x - rb);
        *bb = *bb + step;
      }
  }
  fo_ccache_refresh(dims[mode], jn, r, amat[mode], bmat[mode], cmat[mode]);
  free(d); free(g);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* fp64 evaluation (model.cpp:70-92, evaluation.cpp:10-72).                 */

double fo_predict(int order, const int32_t* ranks, int r, float* const* amat,
                  float* const* bmat, const int32_t* idx) {
  double acc = 0.0;
  for (int c = 0; c < r; ++c) {
    double prod = 1.0;
    for (int n = 0; n < order; ++n) {
      const float* row = amat[n] + (size_t)idx[n] * ranks[n];
      double s = 0.0;
      for (int j = 0; j < ranks[n]; ++j) {
        double t = (double)row[j] * (double)bmat[n][(size_t)j * r + c];
        s = s + t;
      }
      prod = prod * s;
    }
    acc = acc + prod;
  }
  return acc;
}

/* Slab reduction: ceil(n/workers) contiguous entries per worker, each summed
 * in entry order, slabs combined in worker order (evaluation.cpp:13-32).
 * kind 0 = squared residual, 1 = absolute residual. */
static double slab_sum(int order, const int32_t* ranks, int r,
                       float* const* amat, float* const* bmat, int64_t nnz,
                       const int32_t* idx_aos, const float* vals, int workers,
                       int kind) {
  if (workers < 1) workers = 1;
  int64_t chunk = (nnz + workers - 1) / workers;
  double total = 0.0;
  for (int wk = 0; wk < workers; ++wk) {
    int64_t lo = wk * chunk, hi = lo + chunk < nnz ? lo + chunk : nnz;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) {
      double res = (double)vals[i] -
                   fo_predict(order, ranks, r, amat, bmat, idx_aos + i * order);
      s = s + (kind == 0 ? res * res : fabs(res));
    }
    total = total + s;
  }
  return total;
}

double fo_loss(int order, const int32_t* dims, const int32_t* ranks, int r,
               float* const* amat, float* const* bmat, int64_t nnz,
               const int32_t* idx_aos, const float* vals, double reg_a,
               double reg_b, int workers) {
  double data = slab_sum(order, ranks, r, amat, bmat, nnz, idx_aos, vals,
                         workers, 0);
  double reg = 0.0;
  for (int n = 0; n < order; ++n) {
    double sq = 0.0;
    size_t len = (size_t)dims[n] * ranks[n];
    for (size_t i = 0; i < len; ++i) sq = sq + (double)amat[n][i] * amat[n][i];
    reg = reg + reg_a * sq;
  }
  for (int n = 0; n < order; ++n) {
    double sq = 0.0;
    size_t len = (size_t)ranks[n] * r;
    for (size_t i = 0; i < len; ++i) sq = sq + (double)bmat[n][i] * bmat[n][i];
    reg = reg + reg_b * sq;
  }
  return data + reg;
}

void fo_evaluate(int order, const int32_t* ranks, int r, float* const* amat,
                 float* const* bmat, int64_t nnz, const int32_t* idx_aos,
                 const float* vals, int workers, double* rmse, double* mae) {
  double sq = slab_sum(order, ranks, r, amat, bmat, nnz, idx_aos, vals, workers, 0);
  double ab = slab_sum(order, ranks, r, amat, bmat, nnz, idx_aos, vals, workers, 1);
  *rmse = sqrt(sq / (double)nnz);
  *mae = ab / (double)nnz;
}

/* Closed-form per-full-batch plus costs (counters.cpp:486-491). */
void fo_predicted_costs(int order, int m, int r, const int32_t* ranks,
                        int64_t* out4) {
  int64_t n = order, mm_ = m, rr = r, sj = 0;
  for (int k = 0; k < order; ++k) sj += ranks[k];
  out4[0] = (mm_ + rr) * sj;
  out4[1] = mm_ * rr * (sj + n * (n - 2));
  out4[2] = mm_ * rr * sj;
  out4[3] = mm_ * sj;
}
