/*
 * dssync_oracle.c — CPU restatement of the reference's DS-Sync hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may use it, and only as the checker.
 *
 * Parity of this restatement is pinned against the reference itself: the
 * double instantiation is compared bit for bit with the unmodified
 * reference sources compiled by oracle/Makefile into oracle/_ref/ (see
 * tests/test_oracle.py) and against the golden fixtures the reference
 * produced (tests/golden/, made by tests/golden/make_golden.py).
 *
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).  The float instantiation is
 * the same operation sequence in binary32 with every constant rounded once
 * from its double value — the contract the fp32 CUDA path is bit-exact to.
 *
 * Build: gcc -O2 -ffp-contract=off (x86-64 SSE: every + and * rounds
 * separately, like the reference's Release build).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_EDIVERGED 2

/* ---------------- rng.cpp:8-51 ------------------------------------------ */

static uint64_t mix64(uint64_t z) { /* rng.cpp:10-14 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_for_stream(uint64_t seed, uint64_t purpose, uint64_t rank, uint64_t it) { /* rng.cpp:20-26 */
  uint64_t s = mix64(seed + 0x9e3779b97f4a7c15ULL);
  s = mix64(s ^ purpose);
  s = mix64(s ^ rank);
  s = mix64(s ^ it);
  return s;
}

uint64_t orc_next_u64(uint64_t* state) { /* rng.cpp:28-31 */
  *state += 0x9e3779b97f4a7c15ULL;
  return mix64(*state);
}

static double uniform01(uint64_t* st) { /* rng.cpp:33-35 */
  return (double)(orc_next_u64(st) >> 11) * 0x1.0p-53;
}

double orc_gaussian(uint64_t* st) { /* rng.cpp:46-51 */
  const double u1 = 1.0 - uniform01(st);
  const double u2 = uniform01(st);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* n gaussians of stream (seed, purpose, rank, it), from the start. */
void orc_gaussian_stream(uint64_t seed, uint64_t purpose, uint64_t rank, uint64_t it, long n, double* out) {
  uint64_t st = orc_for_stream(seed, purpose, rank, it);
  for (long i = 0; i < n; ++i) out[i] = orc_gaussian(&st);
}

/* ---------------- schedule.cpp:8-54 (+ rectangular extension) ----------- */

int orc_validate_world(int W, int N, int rect) { /* schedule.cpp:8-24 */
  if (W < 1 || N < 1) return ORC_EINVAL;
  if (rect) return (W % N == 0) ? ORC_OK : ORC_EINVAL;
  if ((long)W != (long)N * N && W != N) return ORC_EINVAL;
  return ORC_OK;
}

/* kind: 0 bsp (partition_for, sync.cpp:131-139), 1 ds-sync (make_partition).
 * Square: g(x) = t even ? x / N : x % N (schedule.cpp:45-50).  Rect W = N*K:
 * the same rule, K blocks of N (even) / N combs of K (odd). */
int orc_partition(int W, int N, int rect, int kind, long t, int* members, int* offsets, int* n_groups) {
  if (kind == 0 || W == N) {
    for (int x = 0; x < W; ++x) members[x] = x;
    offsets[0] = 0;
    offsets[1] = W;
    *n_groups = 1;
    return ORC_OK;
  }
  if (orc_validate_world(W, N, rect) != ORC_OK || t < 0) return ORC_EINVAL;
  const int K = W / N;
  const int even = (t % 2 == 0);
  const int groups = even ? K : N;
  int pos = 0;
  for (int g = 0; g < groups; ++g) {
    offsets[g] = pos;
    for (int x = 0; x < W; ++x) {
      const int gx = even ? x / N : x % N;
      if (gx == g) members[pos++] = x;
    }
  }
  offsets[groups] = pos;
  *n_groups = groups;
  return ORC_OK;
}

/* ---------------- optimizer constants ----------------------------------- */

typedef struct {
  double momentum, beta1, beta2, epsilon, weight_decay;
} orc_hparams; /* optim.hpp:16-23 (alpha passed separately) */

/* Generates the per-type restatement.  T = double reproduces optim.cpp:46-98,
 * param.cpp:42-53 and comm.cpp:78-123 bit for bit; T = float is the same
 * sequence in binary32 with constants rounded once from double. */
#define ORC_DEFINE(T, SUF, SQRT, ISFIN)                                                          \
  typedef struct {                                                                              \
    T a, wd, mom, b1, omb1, b2, omb2, eps, awd;                                                 \
  } consts_##SUF;                                                                               \
                                                                                                \
  static consts_##SUF make_consts_##SUF(const orc_hparams* h, double alpha) {                   \
    consts_##SUF c;                                                                             \
    c.a = (T)alpha;                                                                             \
    c.wd = (T)h->weight_decay;                                                                  \
    c.mom = (T)h->momentum;                                                                     \
    c.b1 = (T)h->beta1;                                                                         \
    c.omb1 = (T)(1.0 - h->beta1);                                                               \
    c.b2 = (T)h->beta2;                                                                         \
    c.omb2 = (T)(1.0 - h->beta2);                                                               \
    c.eps = (T)h->epsilon;                                                                      \
    c.awd = (T)(alpha * h->weight_decay);                                                       \
    return c;                                                                                   \
  }                                                                                             \
                                                                                                \
  /* apply_step on one worker row (optim.cpp:46-98); returns 0 when finite. */                  \
  static int step_row_##SUF(int opt, const consts_##SUF* c, long step_count, const orc_hparams* h, \
                            long d, T* w, const T* g, long g_stride_zero, T* m1, T* m2) {       \
    int ok = 1;                                                                                 \
    const T bc1 = (T)(1.0 - pow(h->beta1, (double)(step_count + 1)));                           \
    const T bc2 = (T)(1.0 - pow(h->beta2, (double)(step_count + 1)));                           \
    (void)g_stride_zero;                                                                        \
    for (long i = 0; i < d; ++i) {                                                              \
      const T wi = w[i];                                                                        \
      T out;                                                                                    \
      if (opt == 0) { /* optim.cpp:56-61 */                                                     \
        const T ge = g[i] + c->wd * wi;                                                         \
        out = wi - c->a * ge;                                                                   \
      } else if (opt == 1) { /* optim.cpp:63-70 */                                              \
        const T ge = g[i] + c->wd * wi;                                                         \
        m1[i] = c->mom * m1[i] + ge;                                                            \
        out = wi - c->a * m1[i];                                                                \
      } else { /* optim.cpp:72-91 */                                                            \
        const T ge = (opt == 2) ? g[i] + c->wd * wi : g[i];                                     \
        m1[i] = c->b1 * m1[i] + c->omb1 * ge;                                                   \
        m2[i] = c->b2 * m2[i] + c->omb2 * ge * ge;                                              \
        const T mhat = m1[i] / bc1;                                                             \
        const T vhat = m2[i] / bc2;                                                             \
        out = wi - c->a * mhat / (SQRT(vhat) + c->eps);                                         \
        if (opt == 3) out -= c->awd * wi;                                                       \
      }                                                                                         \
      w[i] = out;                                                                               \
      if (!ISFIN(out)) ok = 0;                                                                  \
    }                                                                                           \
    return ok ? 0 : 1;                                                                          \
  }                                                                                             \
                                                                                                \
  /* mean_of over member rows in ascending order (param.cpp:42-53 /                            \
   * comm.cpp:96-110), written to every member.  Returns 0 when finite. */                      \
  static int fold_group_##SUF(long d, const int* mem, int m, T* base, long ld, T* acc) {       \
    memcpy(acc, base + (long)mem[0] * ld, sizeof(T) * (size_t)d);                               \
    for (int k = 1; k < m; ++k) {                                                               \
      const T* x = base + (long)mem[k] * ld;                                                    \
      for (long i = 0; i < d; ++i) acc[i] += x[i];                                              \
    }                                                                                           \
    int ok = 1;                                                                                 \
    if (m > 1) { /* comm.cpp:85-88: a lone member is returned unscaled */                       \
      const T inv = (T)(1.0 / (double)m);                                                       \
      for (long i = 0; i < d; ++i) {                                                            \
        acc[i] *= inv;                                                                          \
        if (!ISFIN(acc[i])) ok = 0;                                                             \
      }                                                                                         \
    }                                                                                           \
    for (int k = 0; k < m; ++k) memcpy(base + (long)mem[k] * ld, acc, sizeof(T) * (size_t)d);   \
    return ok ? 0 : 1;                                                                          \
  }                                                                                             \
                                                                                                \
  /* One DS-Sync iteration on [W][d] rows (sync.cpp:347-374): every worker                      \
   * steps (ascending rank), then every group averages.  err_rank/err_phase                     \
   * report the first failure the reference would throw. */                                    \
  int orc_ds_step_##SUF(int W, int N, int rect, long d, long t, int opt, const orc_hparams* h,  \
                        double alpha, const long* step_counts, T* w, const T* g, T* m1, T* m2,  \
                        int* err_rank, int* err_phase) {                                        \
    int* members = (int*)malloc(sizeof(int) * (size_t)W);                                       \
    int* offsets = (int*)malloc(sizeof(int) * (size_t)(W + 1));                                 \
    T* acc = (T*)malloc(sizeof(T) * (size_t)d);                                                 \
    int ng = 0, rc = ORC_OK;                                                                    \
    const consts_##SUF c = make_consts_##SUF(h, alpha);                                         \
    *err_rank = -1;                                                                             \
    *err_phase = -1;                                                                            \
    if (orc_partition(W, N, rect, 1, t, members, offsets, &ng) != ORC_OK) {                     \
      rc = ORC_EINVAL;                                                                          \
      goto done;                                                                                \
    }                                                                                           \
    for (int k = 0; k < W; ++k) {                                                               \
      const long r = (long)k * d;                                                               \
      if (step_row_##SUF(opt, &c, step_counts[k], h, d, w + r, g + r, 0, m1 ? m1 + r : 0,       \
                         m2 ? m2 + r : 0) && rc == ORC_OK) {                                    \
        rc = ORC_EDIVERGED;                                                                     \
        *err_rank = k;                                                                          \
        *err_phase = 0;                                                                         \
      }                                                                                         \
    }                                                                                           \
    if (rc != ORC_OK) goto done;                                                                \
    for (int gi = 0; gi < ng; ++gi) {                                                           \
      const int* mem = members + offsets[gi];                                                   \
      if (fold_group_##SUF(d, mem, offsets[gi + 1] - offsets[gi], w, d, acc) && rc == ORC_OK) { \
        rc = ORC_EDIVERGED;                                                                     \
        *err_rank = mem[0];                                                                     \
        *err_phase = 1;                                                                         \
      }                                                                                         \
    }                                                                                           \
  done:                                                                                         \
    free(members);                                                                              \
    free(offsets);                                                                              \
    free(acc);                                                                                  \
    return rc;                                                                                  \
  }                                                                                             \
                                                                                                \
  /* sync_round (sync.cpp:268-282): group averaging only. */                                    \
  int orc_sync_round_##SUF(int W, int N, int rect, int kind, long d, long t, T* w, int* err_rank) { \
    int* members = (int*)malloc(sizeof(int) * (size_t)W);                                       \
    int* offsets = (int*)malloc(sizeof(int) * (size_t)(W + 1));                                 \
    T* acc = (T*)malloc(sizeof(T) * (size_t)d);                                                 \
    int ng = 0, rc = ORC_OK;                                                                    \
    *err_rank = -1;                                                                             \
    if (orc_partition(W, N, rect, kind, t, members, offsets, &ng) != ORC_OK) {                  \
      rc = ORC_EINVAL;                                                                          \
    } else {                                                                                    \
      for (int gi = 0; gi < ng; ++gi) {                                                         \
        const int* mem = members + offsets[gi];                                                 \
        if (fold_group_##SUF(d, mem, offsets[gi + 1] - offsets[gi], w, d, acc) && rc == ORC_OK) { \
          rc = ORC_EDIVERGED;                                                                   \
          *err_rank = mem[0];                                                                   \
        }                                                                                       \
      }                                                                                         \
    }                                                                                           \
    free(members);                                                                              \
    free(offsets);                                                                              \
    free(acc);                                                                                  \
    return rc;                                                                                  \
  }                                                                                             \
                                                                                                \
  /* One BSP iteration (sync.cpp:375-428): mean gradient over all W in                          \
   * ascending order, then every worker steps with it. */                                       \
  int orc_bsp_step_##SUF(int W, long d, long t, int opt, const orc_hparams* h, double alpha,    \
                         const long* step_counts, T* w, const T* g, T* m1, T* m2, int* err_rank, \
                         int* err_phase) {                                                      \
    T* gm = (T*)malloc(sizeof(T) * (size_t)d);                                                  \
    int rc = ORC_OK;                                                                            \
    const consts_##SUF c = make_consts_##SUF(h, alpha);                                         \
    (void)t;                                                                                    \
    *err_rank = -1;                                                                             \
    *err_phase = -1;                                                                            \
    memcpy(gm, g, sizeof(T) * (size_t)d);                                                       \
    for (int k = 1; k < W; ++k) {                                                               \
      for (long i = 0; i < d; ++i) gm[i] += g[(long)k * d + i];                                 \
    }                                                                                           \
    if (W > 1) {                                                                                \
      const T inv = (T)(1.0 / (double)W);                                                       \
      for (long i = 0; i < d; ++i) {                                                            \
        gm[i] *= inv;                                                                           \
        if (!ISFIN(gm[i]) && rc == ORC_OK) {                                                    \
          rc = ORC_EDIVERGED;                                                                   \
          *err_rank = 0;                                                                        \
          *err_phase = 0;                                                                       \
        }                                                                                       \
      }                                                                                         \
    }                                                                                           \
    if (rc == ORC_OK) {                                                                         \
      for (int k = 0; k < W; ++k) {                                                             \
        const long r = (long)k * d;                                                             \
        if (step_row_##SUF(opt, &c, step_counts[k], h, d, w + r, gm, 0, m1 ? m1 + r : 0,        \
                           m2 ? m2 + r : 0) && rc == ORC_OK) {                                  \
          rc = ORC_EDIVERGED;                                                                   \
          *err_rank = k;                                                                        \
          *err_phase = 1;                                                                       \
        }                                                                                       \
      }                                                                                         \
    }                                                                                           \
    free(gm);                                                                                   \
    return rc;                                                                                  \
  }                                                                                             \
                                                                                                \
  /* apply_step for every worker with its own gradient, no averaging. */                        \
  int orc_apply_step_##SUF(int W, long d, int opt, const orc_hparams* h, double alpha,          \
                           const long* step_counts, T* w, const T* g, T* m1, T* m2, int* err_rank) { \
    const consts_##SUF c = make_consts_##SUF(h, alpha);                                         \
    int rc = ORC_OK;                                                                            \
    *err_rank = -1;                                                                             \
    for (int k = 0; k < W; ++k) {                                                               \
      const long r = (long)k * d;                                                               \
      if (step_row_##SUF(opt, &c, step_counts[k], h, d, w + r, g + r, 0, m1 ? m1 + r : 0,       \
                         m2 ? m2 + r : 0) && rc == ORC_OK) {                                    \
        rc = ORC_EDIVERGED;                                                                     \
        *err_rank = k;                                                                          \
      }                                                                                         \
    }                                                                                           \
    return rc;                                                                                  \
  }                                                                                             \
                                                                                                \
  /* Isotropic quadratic gradient (problems.cpp:173-193 with A = mu*I,                          \
   * problems.cpp:134-136): the dense matvec over exact zeros is +0 + mu*x_i;                   \
   * noise (sigma/sqrt(d)) * gaussian_i of stream (seed, kGradientNoise,                        \
   * rank, t) computed in double, rounded once to T. */                                         \
  void orc_quadratic_grad_##SUF(int nrows, int first_rank, long d, long t, uint64_t seed,       \
                                double mu, double sigma, const T* w, const T* wstar, T* g) {    \
    const double scale = sigma / sqrt((double)d);                                               \
    const T muT = (T)mu;                                                                        \
    for (int k = 0; k < nrows; ++k) {                                                           \
      uint64_t st = orc_for_stream(seed, 0xa0761d6478bd642fULL, (uint64_t)(first_rank + k),     \
                                   (uint64_t)t);                                                \
      for (long i = 0; i < d; ++i) {                                                            \
        T gi = (T)0 + muT * (w[(long)k * d + i] - wstar[i]);                                    \
        if (sigma > 0.0) gi += (T)(scale * orc_gaussian(&st));                                  \
        g[(long)k * d + i] = gi;                                                                \
      }                                                                                         \
    }                                                                                           \
  }

ORC_DEFINE(double, f64, sqrt, isfinite)
ORC_DEFINE(float, f32, sqrtf, isfinite)

/* w* (problems.cpp:157-159) and w0 = w* + sqrt(delta0) * u, u the normalised
 * gaussian vector of stream (seed, kInitParams, 0, 0) (problems.cpp:106-113,
 * 161-165), in double. */
void orc_quadratic_init_f64(uint64_t seed, long d, double delta0, double* wstar, double* w0) {
  orc_gaussian_stream(seed, 0x9e3779b97f4a7c15ULL, 1, 0, d, wstar);
  double* u = (double*)malloc(sizeof(double) * (size_t)d);
  orc_gaussian_stream(seed, 0xbf58476d1ce4e5b9ULL, 0, 0, d, u);
  double acc = 0.0;
  for (long i = 0; i < d; ++i) acc += u[i] * u[i];
  const double n = sqrt(acc);
  for (long i = 0; i < d; ++i) u[i] /= n;
  const double r = sqrt(delta0);
  for (long i = 0; i < d; ++i) w0[i] = wstar[i] + r * u[i];
  free(u);
}
