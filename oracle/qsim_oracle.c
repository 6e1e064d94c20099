/* qsim_oracle.c -- CPU restatement of the reference's state-vector hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see qsim_oracle.h).  Serial C, complex arithmetic
 * through C99 double _Complex so the expression structure follows the
 * reference's std::complex<double> code; compiled with GNU C semantics
 * (-ffp-contract=fast, as the reference's g++ build).  Every function cites
 * the reference lines it restates (relative to proj/include/qforge/).
 */
#include "qsim_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double _Complex cplx;
static const double kPi = 3.14159265358979323846;

static inline cplx ld(const double* a, uint64_t i) { return CMPLX(a[2 * i], a[2 * i + 1]); }
static inline void st(double* a, uint64_t i, cplx v) {
  a[2 * i] = creal(v);
  a[2 * i + 1] = cimag(v);
}
/* std::norm(a) = re*re + im*im; g++ -O3 contracts it to fma(re, re, im*im). */
static inline double norm2(cplx a) {
  const double re = creal(a), im = cimag(a);
  return re * re + im * im;
}

/* ------------------------------------------------------------------ rng.hpp */
uint64_t qo_splitmix64(uint64_t x) { /* rng.hpp:9-14 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* std::mt19937_64 (the engine behind Rng, rng.hpp:20-46), standard parameters. */
void qo_rng_seed(qo_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}
void qo_rng_derive(qo_rng* r, uint64_t seed, uint64_t index) { /* rng.hpp:26-28 */
  qo_rng_seed(r, qo_splitmix64(seed ^ qo_splitmix64(index + 1)));
}
uint64_t qo_rng_next(qo_rng* r) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & upper) | (r->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}
double qo_rng_uniform(qo_rng* r) { return (double)(qo_rng_next(r) >> 11) * 0x1.0p-53; } /* :33-35 */
uint64_t qo_rng_below(qo_rng* r, uint64_t k) { return qo_rng_next(r) % k; }           /* :42 */
void qo_uniforms(uint64_t seed, uint64_t count, double* out) {
  qo_rng r;
  qo_rng_seed(&r, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = qo_rng_uniform(&r);
}

/* ---------------------------------------------------------------- gates.hpp */
static int target_arity(int kind) {
  switch (kind) {
    case QO_CNOT: case QO_CZ: case QO_SWAP: return 2;
    case QO_TOFFOLI: return 3;
    default: return 1;
  }
}

/* standard_gate_matrix (gates.hpp:15-76) into row-major m (dim x dim). */
static int standard_matrix(int kind, const double* p, cplx* m) {
  const cplx i1 = CMPLX(0.0, 1.0);
  int dim = 1 << target_arity(kind);
  for (int k = 0; k < dim * dim; ++k) m[k] = 0;
  if (dim == 2) {
    switch (kind) {
      case QO_I: m[0] = 1; m[3] = 1; break;
      case QO_X: m[1] = 1; m[2] = 1; break;
      case QO_Y: m[1] = -i1; m[2] = i1; break;
      case QO_Z: m[0] = 1; m[3] = -1; break;
      case QO_H: {
        double s = 1.0 / sqrt(2.0);
        m[0] = s; m[1] = s; m[2] = s; m[3] = -s;
        break;
      }
      case QO_S: m[0] = 1; m[3] = i1; break;
      case QO_T: m[0] = 1; m[3] = cexp(i1 * (kPi / 4)); break;
      case QO_RX: {
        double c = cos(p[0] / 2), s = sin(p[0] / 2);
        m[0] = c; m[1] = -i1 * s; m[2] = -i1 * s; m[3] = c;
        break;
      }
      case QO_RY: {
        double c = cos(p[0] / 2), s = sin(p[0] / 2);
        m[0] = c; m[1] = -s; m[2] = s; m[3] = c;
        break;
      }
      case QO_RZ:
        m[0] = cexp(-i1 * (p[0] / 2)); m[3] = cexp(i1 * (p[0] / 2));
        break;
      case QO_U3: {
        double th = p[0], ph = p[1], la = p[2];
        double c = cos(th / 2), s = sin(th / 2);
        m[0] = c; m[1] = -cexp(i1 * la) * s; m[2] = cexp(i1 * ph) * s; m[3] = cexp(i1 * (la + ph)) * c;
        break;
      }
      default: return -1;
    }
  } else {
    for (int k = 0; k < dim; ++k) m[k * dim + k] = 1;
    switch (kind) {
      case QO_CNOT: m[2 * 4 + 2] = 0; m[3 * 4 + 3] = 0; m[2 * 4 + 3] = 1; m[3 * 4 + 2] = 1; break;
      case QO_CZ: m[3 * 4 + 3] = -1; break;
      case QO_SWAP: m[1 * 4 + 1] = 0; m[2 * 4 + 2] = 0; m[1 * 4 + 2] = 1; m[2 * 4 + 1] = 1; break;
      case QO_TOFFOLI: m[6 * 8 + 6] = 0; m[7 * 8 + 7] = 0; m[6 * 8 + 7] = 1; m[7 * 8 + 6] = 1; break;
      default: return -1;
    }
  }
  return dim;
}

/* base_matrix (gates.hpp:91-97): custom or named matrix, adjoint if dagger. */
static int base_matrix(const qo_gate* g, cplx* m) {
  int dim;
  if (g->kind == QO_CUSTOM) {
    if (!g->matrix || g->num_targets == 0 || g->num_targets > 8) return -1;
    dim = 1 << g->num_targets;
    for (int k = 0; k < dim * dim; ++k) m[k] = CMPLX(g->matrix[2 * k], g->matrix[2 * k + 1]);
  } else {
    dim = standard_matrix(g->kind, g->params, m);
    if (dim < 0) return -1;
  }
  if (g->dagger) {
    for (int r = 0; r < dim; ++r)
      for (int c = r; c < dim; ++c) {
        cplx a = m[r * dim + c], b = m[c * dim + r];
        m[r * dim + c] = conj(b);
        m[c * dim + r] = conj(a);
      }
  }
  return dim;
}

int qo_base_matrix(const qo_gate* g, double* out) {
  cplx* m = malloc(sizeof(cplx) * 65536);
  int dim = base_matrix(g, m);
  if (dim > 0)
    for (int k = 0; k < dim * dim; ++k) { out[2 * k] = creal(m[k]); out[2 * k + 1] = cimag(m[k]); }
  free(m);
  return dim;
}

/* linalg.hpp:28-32: max |M^H M - I| <= tol */
static int is_unitary(const cplx* m, int dim, double tol) {
  double worst = 0;
  for (int i = 0; i < dim; ++i)
    for (int j = 0; j < dim; ++j) {
      cplx s = 0;
      for (int k = 0; k < dim; ++k) s += conj(m[k * dim + i]) * m[k * dim + j];
      if (i == j) s -= 1;
      double a = cabs(s);
      if (a > worst) worst = a;
    }
  return worst <= tol;
}

/* ---------------------------------------------------------- statevector.hpp */
/* GroupIndexer (statevector.hpp:42-64): insert zero bits at the sorted
 * reserved positions, then OR in the control mask. */
typedef struct {
  uint32_t slots[64];
  uint32_t nslots;
  uint64_t force_mask;
} indexer;

static void ix_init(indexer* ix) { ix->nslots = 0; ix->force_mask = 0; }
static void ix_target(indexer* ix, uint32_t q) { ix->slots[ix->nslots++] = q; }
static void ix_control(indexer* ix, uint32_t q) {
  ix->slots[ix->nslots++] = q;
  ix->force_mask |= 1ULL << q;
}
static void ix_finish(indexer* ix) {
  for (uint32_t i = 1; i < ix->nslots; ++i)
    for (uint32_t j = i; j > 0 && ix->slots[j - 1] > ix->slots[j]; --j) {
      uint32_t t = ix->slots[j]; ix->slots[j] = ix->slots[j - 1]; ix->slots[j - 1] = t;
    }
}
static inline uint64_t ix_groups(const indexer* ix, uint32_t n) { return 1ULL << (n - ix->nslots); }
static inline uint64_t ix_base(const indexer* ix, uint64_t g) {
  uint64_t x = g;
  for (uint32_t s = 0; s < ix->nslots; ++s) {
    uint32_t pos = ix->slots[s];
    uint64_t low = x & ((1ULL << pos) - 1);
    x = ((x >> pos) << (pos + 1)) | low;
  }
  return x | ix->force_mask;
}

void qo_init_zero(double* amps, uint32_t n) { /* statevector.hpp:136-141 */
  memset(amps, 0, sizeof(double) * 2 * (1ULL << n));
  amps[0] = 1.0;
}

void qo_apply_1q(double* amps, uint32_t n, uint32_t q, const double mm[8], const uint32_t* ctrls,
                 uint32_t nc) { /* statevector.hpp:268-290 */
  indexer ix;
  ix_init(&ix);
  ix_target(&ix, q);
  for (uint32_t c = 0; c < nc; ++c) ix_control(&ix, ctrls[c]);
  ix_finish(&ix);
  const cplx m0 = CMPLX(mm[0], mm[1]), m1 = CMPLX(mm[2], mm[3]);
  const cplx m2 = CMPLX(mm[4], mm[5]), m3 = CMPLX(mm[6], mm[7]);
  const uint64_t bit = 1ULL << q, groups = ix_groups(&ix, n);
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t i0 = ix_base(&ix, g), i1 = i0 | bit;
    const cplx a = ld(amps, i0), b = ld(amps, i1);
    st(amps, i0, m0 * a + m1 * b);
    st(amps, i1, m2 * a + m3 * b);
  }
}

void qo_apply_diag(double* amps, uint32_t n, uint32_t q, const double d[4], const uint32_t* ctrls,
                   uint32_t nc) { /* statevector.hpp:292-319 */
  const cplx d0 = CMPLX(d[0], d[1]), d1 = CMPLX(d[2], d[3]);
  indexer ix;
  ix_init(&ix);
  const int skip_zero = (d0 == 1.0);
  if (skip_zero) ix_control(&ix, q);
  else ix_target(&ix, q);
  for (uint32_t c = 0; c < nc; ++c) ix_control(&ix, ctrls[c]);
  ix_finish(&ix);
  const uint64_t bit = 1ULL << q, groups = ix_groups(&ix, n);
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t i0 = ix_base(&ix, g);
    if (skip_zero) {
      st(amps, i0, ld(amps, i0) * d1);
    } else {
      st(amps, i0, ld(amps, i0) * d0);
      st(amps, i0 | bit, ld(amps, i0 | bit) * d1);
    }
  }
}

void qo_apply_flip(double* amps, uint32_t n, uint32_t q, const uint32_t* ctrls, uint32_t nc) {
  /* statevector.hpp:321-339 */
  indexer ix;
  ix_init(&ix);
  ix_target(&ix, q);
  for (uint32_t c = 0; c < nc; ++c) ix_control(&ix, ctrls[c]);
  ix_finish(&ix);
  const uint64_t bit = 1ULL << q, groups = ix_groups(&ix, n);
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t i0 = ix_base(&ix, g);
    const cplx t = ld(amps, i0);
    st(amps, i0, ld(amps, i0 | bit));
    st(amps, i0 | bit, t);
  }
}

void qo_apply_swap2(double* amps, uint32_t n, uint32_t a, uint32_t b, const uint32_t* ctrls,
                    uint32_t nc) { /* statevector.hpp:341-361 */
  indexer ix;
  ix_init(&ix);
  ix_target(&ix, a);
  ix_target(&ix, b);
  for (uint32_t c = 0; c < nc; ++c) ix_control(&ix, ctrls[c]);
  ix_finish(&ix);
  const uint64_t ba = 1ULL << a, bb = 1ULL << b, groups = ix_groups(&ix, n);
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t base = ix_base(&ix, g);
    const cplx t = ld(amps, base | ba);
    st(amps, base | ba, ld(amps, base | bb));
    st(amps, base | bb, t);
  }
}

int qo_apply_matrix(double* amps, uint32_t n, const uint32_t* targets, uint32_t k, const double* m,
                    const uint32_t* ctrls, uint32_t nc) { /* statevector.hpp:363-467 */
  if (k + nc > n) return -1;
  if (k == 1) {
    qo_apply_1q(amps, n, targets[0], m, ctrls, nc);
    return 0;
  }
  indexer ix;
  ix_init(&ix);
  for (uint32_t t = 0; t < k; ++t) ix_target(&ix, targets[t]);
  for (uint32_t c = 0; c < nc; ++c) ix_control(&ix, ctrls[c]);
  ix_finish(&ix);
  const uint64_t ldim = 1ULL << k;
  uint64_t* offset = calloc(ldim, sizeof(uint64_t));
  for (uint64_t p = 0; p < ldim; ++p)
    for (uint32_t b = 0; b < k; ++b)
      if (p & (1ULL << b)) offset[p] |= 1ULL << targets[k - 1 - b];
  /* planar column-major coefficients (:395-402) */
  double* mre = malloc(sizeof(double) * ldim * ldim);
  double* mim = malloc(sizeof(double) * ldim * ldim);
  for (uint64_t c = 0; c < ldim; ++c)
    for (uint64_t r = 0; r < ldim; ++r) {
      mre[c * ldim + r] = m[2 * (r * ldim + c)];
      mim[c * ldim + r] = m[2 * (r * ldim + c) + 1];
    }
  double* buf = malloc(sizeof(double) * 4 * ldim);
  double *vre = buf, *vim = buf + ldim, *wre = buf + 2 * ldim, *wim = buf + 3 * ldim;
  const uint64_t groups = ix_groups(&ix, n);
  for (uint64_t g = 0; g < groups; ++g) {
    const uint64_t base = ix_base(&ix, g);
    for (uint64_t p = 0; p < ldim; ++p) {
      vre[p] = amps[2 * (base + offset[p])];
      vim[p] = amps[2 * (base + offset[p]) + 1];
      wre[p] = 0.0;
      wim[p] = 0.0;
    }
    for (uint64_t c = 0; c < ldim; ++c) {
      const double xr = vre[c], xi = vim[c];
      const double* col_re = mre + c * ldim;
      const double* col_im = mim + c * ldim;
      for (uint64_t r = 0; r < ldim; ++r) {
        wre[r] += col_re[r] * xr - col_im[r] * xi;
        wim[r] += col_re[r] * xi + col_im[r] * xr;
      }
    }
    for (uint64_t p = 0; p < ldim; ++p) {
      amps[2 * (base + offset[p])] = wre[p];
      amps[2 * (base + offset[p]) + 1] = wim[p];
    }
  }
  free(buf);
  free(mre);
  free(mim);
  free(offset);
  return 0;
}

int qo_apply_gate(double* amps, uint32_t n, const qo_gate* g) { /* statevector.hpp:469-538 */
  const cplx i1 = CMPLX(0.0, 1.0);
  uint32_t cs[48];
  uint32_t nc = g->num_controls;
  for (uint32_t c = 0; c < nc; ++c) cs[c] = g->controls[c];
  const uint32_t* t = g->targets;
  switch (g->kind) {
    case QO_I: return 0;
    case QO_X: qo_apply_flip(amps, n, t[0], cs, nc); return 0;
    case QO_CNOT: cs[nc++] = t[0]; qo_apply_flip(amps, n, t[1], cs, nc); return 0;
    case QO_TOFFOLI:
      cs[nc++] = t[0]; cs[nc++] = t[1];
      qo_apply_flip(amps, n, t[2], cs, nc);
      return 0;
    case QO_Z: { double d[4] = {1, 0, -1, 0}; qo_apply_diag(amps, n, t[0], d, cs, nc); return 0; }
    case QO_CZ: {
      double d[4] = {1, 0, -1, 0};
      cs[nc++] = t[0];
      qo_apply_diag(amps, n, t[1], d, cs, nc);
      return 0;
    }
    case QO_S: {
      cplx d1 = g->dagger ? -i1 : i1;
      double d[4] = {1, 0, creal(d1), cimag(d1)};
      qo_apply_diag(amps, n, t[0], d, cs, nc);
      return 0;
    }
    case QO_T: {
      cplx dd = cexp(i1 * (kPi / 4));
      if (g->dagger) dd = conj(dd);
      double d[4] = {1, 0, creal(dd), cimag(dd)};
      qo_apply_diag(amps, n, t[0], d, cs, nc);
      return 0;
    }
    case QO_RZ: {
      double th = g->dagger ? -g->params[0] : g->params[0];
      cplx d0 = cexp(-i1 * (th / 2)), d1 = cexp(i1 * (th / 2));
      double d[4] = {creal(d0), cimag(d0), creal(d1), cimag(d1)};
      qo_apply_diag(amps, n, t[0], d, cs, nc);
      return 0;
    }
    case QO_SWAP: qo_apply_swap2(amps, n, t[0], t[1], cs, nc); return 0;
    case QO_Y: case QO_H: case QO_RX: case QO_RY: case QO_U3: {
      cplx m[4];
      base_matrix(g, m);
      double mm[8];
      for (int k = 0; k < 4; ++k) { mm[2 * k] = creal(m[k]); mm[2 * k + 1] = cimag(m[k]); }
      qo_apply_1q(amps, n, t[0], mm, cs, nc);
      return 0;
    }
    case QO_CUSTOM: {
      if (!g->matrix || g->num_targets == 0 || g->num_targets > 8) return -1;
      int dim = 1 << g->num_targets;
      cplx* m = malloc(sizeof(cplx) * dim * dim);
      double* mm = malloc(sizeof(double) * 2 * dim * dim);
      for (int k = 0; k < dim * dim; ++k) m[k] = CMPLX(g->matrix[2 * k], g->matrix[2 * k + 1]);
      if (!is_unitary(m, dim, 1e-10)) { free(m); free(mm); return -1; }
      base_matrix(g, m);
      for (int k = 0; k < dim * dim; ++k) { mm[2 * k] = creal(m[k]); mm[2 * k + 1] = cimag(m[k]); }
      int rc = qo_apply_matrix(amps, n, g->targets, g->num_targets, mm, cs, nc);
      free(m);
      free(mm);
      return rc;
    }
  }
  return -1;
}

int qo_apply_gates(double* amps, uint32_t n, const qo_gate* g, uint64_t count) {
  for (uint64_t i = 0; i < count; ++i)
    if (qo_apply_gate(amps, n, &g[i]) != 0) return -1;
  return 0;
}

/* chunked_sum (statevector.hpp:110-130): fixed 4096-element chunks, serial
 * inside a chunk, partials summed in index order. */
static double chunked_norm(const double* amps, uint64_t size, int use_bit, uint64_t bit) {
  const uint64_t chunk = 4096, nchunks = (size + chunk - 1) / chunk;
  double total = 0.0;
  for (uint64_t c = 0; c < nchunks; ++c) {
    const uint64_t lo = c * chunk, hi = lo + chunk < size ? lo + chunk : size;
    double s = 0.0;
    for (uint64_t i = lo; i < hi; ++i) s += (!use_bit || (i & bit)) ? norm2(ld(amps, i)) : 0.0;
    total += s;
  }
  return total;
}
double qo_norm2(const double* amps, uint32_t n) { return chunked_norm(amps, 1ULL << n, 0, 0); }
double qo_prob_one(const double* amps, uint32_t n, uint32_t q) {
  return chunked_norm(amps, 1ULL << n, 1, 1ULL << q);
}

void qo_probs(const double* amps, uint32_t n, const uint32_t* qubits, uint32_t m, double* out) {
  /* statevector.hpp:190-208 */
  memset(out, 0, sizeof(double) * (1ULL << m));
  for (uint64_t i = 0; i < (1ULL << n); ++i) {
    double p = norm2(ld(amps, i));
    if (p == 0.0) continue;
    uint64_t key = 0;
    for (uint32_t b = 0; b < m; ++b)
      if (i & (1ULL << qubits[b])) key |= 1ULL << b;
    out[key] += p;
  }
}

void qo_probs_full(const double* amps, uint32_t n, double* out) { /* :210-215 */
  for (uint64_t i = 0; i < (1ULL << n); ++i) out[i] = norm2(ld(amps, i));
}

int qo_collapse(double* amps, uint32_t n, uint32_t q, int outcome, double prob) { /* :228-247 */
  if (prob <= 0.0) return -2;
  const double inv = 1.0 / sqrt(prob);
  const uint64_t bit = 1ULL << q;
  for (uint64_t i = 0; i < (1ULL << n); ++i) {
    const int one = (i & bit) != 0;
    if (one == (outcome == 1)) st(amps, i, ld(amps, i) * inv);
    else st(amps, i, 0);
  }
  return 0;
}

int qo_measure_collapse(double* amps, uint32_t n, uint32_t q, double u) { /* :219-225 */
  double p1 = qo_prob_one(amps, n, q);
  double p0 = 1.0 - p1;
  int outcome = (u < p0) ? 0 : 1;
  if (qo_collapse(amps, n, q, outcome, outcome ? p1 : p0) != 0) return -2;
  return outcome;
}

double qo_checksum(const double* amps, uint32_t n) { /* bench.hpp:141-148 */
  double sum = 0.0;
  for (uint64_t i = 0; i < (1ULL << n); ++i) sum += norm2(ld(amps, i)) * (double)(i + 1);
  return sum;
}

double qo_sampler_build(const double* amps, uint32_t n, double* cum) { /* statevector.hpp:544-552 */
  double acc = 0.0;
  for (uint64_t i = 0; i < (1ULL << n); ++i) {
    acc += norm2(ld(amps, i));
    cum[i] = acc;
  }
  return acc;
}

uint64_t qo_sampler_draw(const double* cum, uint64_t size, double total, double u) { /* :554-565 */
  const double target = u * total;
  uint64_t lo = 0, hi = size - 1;
  while (lo < hi) {
    uint64_t mid = (lo + hi) / 2;
    if (cum[mid] > target) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

void qo_sample_seeded(const double* amps, uint32_t n, uint64_t seed, uint64_t shots, uint64_t* out) {
  /* simulator.hpp:164-178: sampler over the final state, fresh Rng(seed) */
  const uint64_t size = 1ULL << n;
  double* cum = malloc(sizeof(double) * size);
  double total = qo_sampler_build(amps, n, cum);
  qo_rng r;
  qo_rng_seed(&r, seed);
  for (uint64_t s = 0; s < shots; ++s) out[s] = qo_sampler_draw(cum, size, total, qo_rng_uniform(&r));
  free(cum);
}

double qo_expectation(const double* amps, uint32_t n, const char* letters, const double* coeffs,
                      uint32_t nterms, double* imag_out) { /* variational.hpp:33-54 */
  const uint64_t size = 1ULL << n;
  double* h = malloc(sizeof(double) * 2 * size);
  cplx acc = 0;
  for (uint32_t t = 0; t < nterms; ++t) {
    memcpy(h, amps, sizeof(double) * 2 * size);
    for (uint32_t q = 0; q < n; ++q) {
      char l = letters[(uint64_t)t * n + q];
      if (l == 'I') continue;
      qo_gate g;
      memset(&g, 0, sizeof g);
      g.kind = l == 'X' ? QO_X : l == 'Y' ? QO_Y : QO_Z;
      g.num_targets = 1;
      g.targets[0] = q;
      qo_apply_gate(h, n, &g);
    }
    cplx dot = 0;
    for (uint64_t i = 0; i < size; ++i) dot += conj(ld(amps, i)) * ld(h, i);
    acc += coeffs[t] * dot;
  }
  free(h);
  if (imag_out) *imag_out = cimag(acc);
  return creal(acc);
}

/* ----------------------------------------------------------- generators */
static void mk(qo_gate* g, int kind, uint32_t nt, const uint32_t* t, int np, const double* p) {
  memset(g, 0, sizeof *g);
  g->kind = kind;
  g->num_targets = nt;
  for (uint32_t i = 0; i < nt; ++i) g->targets[i] = t[i];
  for (int i = 0; i < np; ++i) g->params[i] = p[i];
}

uint64_t qo_gen_random_circuit(uint32_t n, uint32_t d, uint64_t seed, qo_gate* out) {
  /* bench.hpp:72-94 */
  uint64_t k = 0;
  qo_rng r;
  qo_rng_seed(&r, seed);
  for (uint32_t layer = 0; layer < d; ++layer) {
    for (uint32_t q = 0; q < n; ++q) {
      const uint64_t axis = qo_rng_below(&r, 3);
      const double angle = qo_rng_uniform(&r) * (2.0 * kPi);
      const int kind = axis == 0 ? QO_RX : axis == 1 ? QO_RY : QO_RZ;
      if (out) mk(&out[k], kind, 1, &q, 1, &angle);
      ++k;
    }
    if (n > 1)
      for (uint32_t i = 0; i < n; ++i) {
        uint32_t t[2] = {(i + 1) % n, i};
        if (out) mk(&out[k], QO_CNOT, 2, t, 0, NULL);
        ++k;
      }
  }
  return k;
}

/* GHZ(n): H(0), CNOT(i, i+1) for i < n-1 (oracle/circuits.hpp). */
uint64_t qo_gen_ghz(uint32_t n, qo_gate* out) {
  uint64_t k = 0;
  uint32_t z = 0;
  if (out) mk(&out[k], QO_H, 1, &z, 0, NULL);
  ++k;
  for (uint32_t i = 0; i + 1 < n; ++i) {
    uint32_t t[2] = {i, i + 1};
    if (out) mk(&out[k], QO_CNOT, 2, t, 0, NULL);
    ++k;
  }
  return k;
}

/* QFT(n) on the basis state |input> (oracle/circuits.hpp): X on the set bits
 * of input, then for j = n-1 .. 0: H(j) and, for k = j-1 .. 0, the controlled
 * phase U3(0, 0, pi / 2^(j-k)) with control k on target j; then SWAP(i, n-1-i).
 * With qubit 0 as the least significant bit this maps |x> to
 * sum_k exp(2 pi i x k / 2^n) |k> / sqrt(2^n). */
uint64_t qo_gen_qft(uint32_t n, uint64_t input_basis, qo_gate* out) {
  uint64_t k = 0;
  for (uint32_t q = 0; q < n; ++q)
    if ((input_basis >> q) & 1ULL) {
      if (out) mk(&out[k], QO_X, 1, &q, 0, NULL);
      ++k;
    }
  for (uint32_t jj = n; jj-- > 0;) {
    if (out) mk(&out[k], QO_H, 1, &jj, 0, NULL);
    ++k;
    for (uint32_t c = jj; c-- > 0;) {
      if (out) {
        double p[3] = {0.0, 0.0, kPi / (double)(1ULL << (jj - c))};
        mk(&out[k], QO_U3, 1, &jj, 3, p);
        out[k].num_controls = 1;
        out[k].controls[0] = c;
      }
      ++k;
    }
  }
  for (uint32_t i = 0; i < n / 2; ++i) {
    uint32_t t[2] = {i, n - 1 - i};
    if (out) mk(&out[k], QO_SWAP, 2, t, 0, NULL);
    ++k;
  }
  return k;
}

/* Hardware-efficient ansatz (oracle/circuits.hpp): per layer RY(theta_q),
 * RZ(phi_q) on every qubit, then CNOT(q, q+1) for q < n-1; angles are
 * Rng(seed).uniform(2 pi) in program order. */
uint64_t qo_gen_hea(uint32_t n, uint32_t layers, uint64_t seed, qo_gate* out) {
  uint64_t k = 0;
  qo_rng r;
  qo_rng_seed(&r, seed);
  for (uint32_t l = 0; l < layers; ++l) {
    for (uint32_t q = 0; q < n; ++q) {
      double a = qo_rng_uniform(&r) * (2.0 * kPi);
      if (out) mk(&out[k], QO_RY, 1, &q, 1, &a);
      ++k;
      double b = qo_rng_uniform(&r) * (2.0 * kPi);
      if (out) mk(&out[k], QO_RZ, 1, &q, 1, &b);
      ++k;
    }
    for (uint32_t q = 0; q + 1 < n; ++q) {
      uint32_t t[2] = {q, q + 1};
      if (out) mk(&out[k], QO_CNOT, 2, t, 0, NULL);
      ++k;
    }
  }
  return k;
}
