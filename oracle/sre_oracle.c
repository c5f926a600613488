/*
 * sre_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the stabilizer Renyi entropy (SRE) of an
 * N-qubit pure state, written from the paper (Sierant, Valles-Muns, Garcia-Saez,
 * "Computing quantum magic of state vectors", arXiv:2601.07824; /root/reference/PAPER.md,
 * cited below as P:<line>).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  It shares no code, header, table or helper with the CUDA product path
 * (paper_2601_07824_b200/csrc); neither includes the other.
 *
 * Three independent evaluations of the same sums, from three readings of the paper:
 *   oracle_brute : Eq. (2) literally -- every <psi|X_a Z_b|psi> by applying Z_b, then X_a,
 *                  to the state vector and taking the overlap.  O(8^N).
 *   oracle_pauli : Eq. (2) over explicit tensor products of the 2x2 matrices I, X, Y, Z
 *                  (no (a,b) parametrisation at all).  O(N 8^N).
 *   oracle_fwht  : Alg. 2 literally -- for each X-string a: beta = X_a psi, v_x = conj(beta_x) alpha_x,
 *                  complex in-place fast Hadamard transform (Eq. (13)), accumulate |chi_b|^{2q}.
 *                  O(N 4^N).                                                    (Alg. 2)
 *
 * Sums layout (all three, and the finaliser):  sums[0..n_alpha-1] = S_{alpha_i} = sum_P t^{alpha_i}
 * with t = |<P>|^2 (reading C2 of DESIGN.md: |chi|^{2q}, as SPEC's design decision),
 * sums[n_alpha] = S_1 = sum_P t (purity, Eq. (14), lost_norm P:1162),
 * sums[n_alpha+1] = sum_P t ln t  (for M_1, the q->1 limit of Eq. (2); 0 ln 0 = 0).
 *
 * Arithmetic: amplitudes are read as double, every product/sum is carried in long double
 * (x87 80-bit), per-X-string sums are combined in ascending a order (deterministic for any
 * thread count).  Integer alpha is raised by repeated multiplication, others by powl.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double R;
typedef struct { R re, im; } C;

static int oracle_is_int(double a) { return a == floor(a) && a >= 1.0 && a <= 64.0; }

/* t^alpha for t >= 0 (t = |<P>|^2). */
static R oracle_pow(R t, double alpha) {
  if (oracle_is_int(alpha)) {
    R r = 1.0L;
    for (int k = 0; k < (int)alpha; k++) r *= t;
    return r;
  }
  if (t == 0.0L) return 0.0L;
  return powl(t, (R)alpha);
}

/* Add the contribution of one expectation value with |<P>|^2 = t to a sums vector. */
static void oracle_accumulate(R* acc, R t, const double* alpha, int n_alpha) {
  for (int i = 0; i < n_alpha; i++) acc[i] += oracle_pow(t, alpha[i]);
  acc[n_alpha] += t;
  if (t > 0.0L) acc[n_alpha + 1] += t * logl(t);
}

static int popcount64(uint64_t v) { int c = 0; while (v) { c += (int)(v & 1u); v >>= 1; } return c; }

/* ---------------------------------------------------------------------------------------------
 * brute: <psi|P_{a,b}|psi> with P_{a,b} = X_a Z_b (Eq. (1)), applied as operators:
 *   (Z_b psi)_x = (-1)^{b.x} psi_x        (Z_b|x> = (-1)^{b.x}|x>)
 *   (X_a phi)_{x xor a} = phi_x           (X_a|x> = |x xor a>)
 *   <psi|X_a Z_b psi> = sum_y conj(psi_y) (X_a Z_b psi)_y
 * psi is interleaved (re, im) doubles of length 2*2^N.  If per_a != NULL it receives, for each
 * a in [a_lo, a_hi), the (n_alpha + 2) sums restricted to that X-string.
 * ------------------------------------------------------------------------------------------- */
int oracle_brute(const double* psi, int N, const double* alpha, int n_alpha,
                 uint64_t a_lo, uint64_t a_hi, double* sums, double* per_a) {
  if (N < 1 || N > 14 || n_alpha < 1 || a_lo > a_hi) return 1;
  const uint64_t D = (uint64_t)1 << N;
  if (a_hi > D) return 1;
  const int m = n_alpha + 2;
  const uint64_t na = a_hi - a_lo;
  R* pa = (R*)calloc((size_t)(na ? na : 1) * m, sizeof(R));
  if (!pa) return 2;
#pragma omp parallel
  {
    C* phi = (C*)malloc(sizeof(C) * D);
    C* chi = (C*)malloc(sizeof(C) * D);
#pragma omp for schedule(dynamic, 1)
    for (int64_t k = 0; k < (int64_t)na; k++) {
      uint64_t a = a_lo + (uint64_t)k;
      R* acc = pa + (size_t)k * m;
      for (uint64_t b = 0; b < D; b++) {
        for (uint64_t x = 0; x < D; x++) {              /* phi = Z_b psi */
          R s = (popcount64(b & x) & 1) ? -1.0L : 1.0L;
          phi[x].re = s * psi[2 * x];
          phi[x].im = s * psi[2 * x + 1];
        }
        for (uint64_t x = 0; x < D; x++) chi[x ^ a] = phi[x];  /* chi = X_a phi */
        C e = {0.0L, 0.0L};
        for (uint64_t y = 0; y < D; y++) {                /* <psi|chi> */
          R pr = psi[2 * y], pi = psi[2 * y + 1];
          e.re += pr * chi[y].re + pi * chi[y].im;
          e.im += pr * chi[y].im - pi * chi[y].re;
        }
        oracle_accumulate(acc, e.re * e.re + e.im * e.im, alpha, n_alpha);
      }
    }
    free(phi);
    free(chi);
  }
  R* tot = (R*)calloc(m, sizeof(R));
  for (uint64_t k = 0; k < na; k++)
    for (int i = 0; i < m; i++) {
      tot[i] += pa[k * m + i];
      if (per_a) per_a[k * m + i] = (double)pa[k * m + i];
    }
  for (int i = 0; i < m; i++) sums[i] = (double)tot[i];
  free(tot);
  free(pa);
  return 0;
}

/* ---------------------------------------------------------------------------------------------
 * pauli: Eq. (2) summed over P = P_1 (x) ... (x) P_N with P_j in {I, X, Y, Z}, each
 * applied as its explicit 2x2 matrix to qubit j (qubit j <-> bit j of the basis index):
 *   I = [[1,0],[0,1]]  X = [[0,1],[1,0]]  Y = [[0,-i],[i,0]]  Z = [[1,0],[0,-1]].
 * <psi|P|psi> is real for Hermitian P; the largest |Im| seen is returned in *max_imag.
 * ------------------------------------------------------------------------------------------- */
int oracle_pauli(const double* psi, int N, const double* alpha, int n_alpha, double* sums,
                 double* max_imag) {
  if (N < 1 || N > 8 || n_alpha < 1) return 1;
  const uint64_t D = (uint64_t)1 << N;
  uint64_t nP = 1;
  for (int j = 0; j < N; j++) nP *= 4;
  const int m = n_alpha + 2;
  /* The four matrices, M[p][row][col] as complex. */
  static const double Mre[4][2][2] = {{{1, 0}, {0, 1}}, {{0, 1}, {1, 0}}, {{0, 0}, {0, 0}}, {{1, 0}, {0, -1}}};
  static const double Mim[4][2][2] = {{{0, 0}, {0, 0}}, {{0, 0}, {0, 0}}, {{0, -1}, {1, 0}}, {{0, 0}, {0, 0}}};
  R* pp = (R*)calloc((size_t)nP * m, sizeof(R));
  R* pim = (R*)calloc((size_t)nP, sizeof(R));
#pragma omp parallel
  {
    C* cur = (C*)malloc(sizeof(C) * D);
    C* nxt = (C*)malloc(sizeof(C) * D);
#pragma omp for schedule(dynamic, 4)
    for (int64_t code = 0; code < (int64_t)nP; code++) {
      for (uint64_t x = 0; x < D; x++) { cur[x].re = psi[2 * x]; cur[x].im = psi[2 * x + 1]; }
      uint64_t c = (uint64_t)code;
      for (int j = 0; j < N; j++) {
        int p = (int)(c & 3u);
        c >>= 2;
        for (uint64_t x = 0; x < D; x++) {              /* nxt = (1 (x) .. M_p on qubit j .. (x) 1) cur */
          int row = (int)((x >> j) & 1u);
          uint64_t x0 = x & ~((uint64_t)1 << j), x1 = x0 | ((uint64_t)1 << j);
          R a_re = Mre[p][row][0], a_im = Mim[p][row][0];
          R b_re = Mre[p][row][1], b_im = Mim[p][row][1];
          nxt[x].re = a_re * cur[x0].re - a_im * cur[x0].im + b_re * cur[x1].re - b_im * cur[x1].im;
          nxt[x].im = a_re * cur[x0].im + a_im * cur[x0].re + b_re * cur[x1].im + b_im * cur[x1].re;
        }
        C* t = cur; cur = nxt; nxt = t;
      }
      C e = {0.0L, 0.0L};
      for (uint64_t y = 0; y < D; y++) {                  /* <psi|P psi> */
        R pr = psi[2 * y], pi = psi[2 * y + 1];
        e.re += pr * cur[y].re + pi * cur[y].im;
        e.im += pr * cur[y].im - pi * cur[y].re;
      }
      oracle_accumulate(pp + (size_t)code * m, e.re * e.re, alpha, n_alpha);
      pim[code] = fabsl(e.im);
    }
    free(cur);
    free(nxt);
  }
  R tot[18] = {0};
  R mi = 0.0L;
  for (uint64_t k = 0; k < nP; k++) {
    for (int i = 0; i < m; i++) tot[i] += pp[k * m + i];
    if (pim[k] > mi) mi = pim[k];
  }
  for (int i = 0; i < m; i++) sums[i] = (double)tot[i];
  if (max_imag) *max_imag = (double)mi;
  free(pp);
  free(pim);
  return 0;
}

/* ---------------------------------------------------------------------------------------------
 * fwht: Algorithm 2.  For each X-string a in [a_lo, a_hi):
 *   beta_x = (X_a psi)_x = psi_{x xor a}            (line 3, |psi'> = X_a |psi>)
 *   v_x = conj(beta_x) * alpha_x, alpha_x = psi_x    (line 4, Eq. (12))
 *   chi = H_2^{(x)N} v, unnormalised H_2 = [[1,1],[1,-1]], in place (line 5, Eq. (13))
 *   S_q += sum_b |chi_b|^{2q}                        (line 6, modulus reading C2)
 * The Gray-code stepping of lines 7-8 only changes the order in which a is visited (reading C11).
 * per_a (optional) receives the (n_alpha+2) sums of each X-string; chi_out (optional, only when
 * a_hi - a_lo == 1) receives the complex chi_b, b = 0 .. 2^N-1, interleaved as doubles.
 * ------------------------------------------------------------------------------------------- */
int oracle_fwht(const double* psi, int N, const double* alpha, int n_alpha,
                uint64_t a_lo, uint64_t a_hi, double* sums, double* per_a, double* chi_out) {
  if (N < 1 || N > 26 || n_alpha < 1 || n_alpha > 16 || a_lo > a_hi) return 1;
  const uint64_t D = (uint64_t)1 << N;
  if (a_hi > D) return 1;
  const int m = n_alpha + 2;
  const uint64_t na = a_hi - a_lo;
  R* pa = (R*)calloc((size_t)(na ? na : 1) * m, sizeof(R));
  if (!pa) return 2;
  int err = 0;
#pragma omp parallel
  {
    C* v = (C*)malloc(sizeof(C) * D);
    if (!v) {
#pragma omp atomic write
      err = 2;
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t k = 0; k < (int64_t)na; k++) {
      if (!v) continue;
      uint64_t a = a_lo + (uint64_t)k;
      for (uint64_t x = 0; x < D; x++) {
        R br = psi[2 * (x ^ a)], bi = psi[2 * (x ^ a) + 1];   /* beta_x */
        R ar = psi[2 * x], ai = psi[2 * x + 1];               /* alpha_x */
        v[x].re = br * ar + bi * ai;                          /* conj(beta) * alpha */
        v[x].im = br * ai - bi * ar;
      }
      for (uint64_t h = 1; h < D; h <<= 1)                    /* fast Hadamard transform */
        for (uint64_t i = 0; i < D; i += 2 * h)
          for (uint64_t j = i; j < i + h; j++) {
            C u = v[j], w = v[j + h];
            v[j].re = u.re + w.re; v[j].im = u.im + w.im;
            v[j + h].re = u.re - w.re; v[j + h].im = u.im - w.im;
          }
      R* acc = pa + (size_t)k * m;
      for (uint64_t b = 0; b < D; b++) oracle_accumulate(acc, v[b].re * v[b].re + v[b].im * v[b].im, alpha, n_alpha);
      if (chi_out && na == 1)
        for (uint64_t b = 0; b < D; b++) { chi_out[2 * b] = (double)v[b].re; chi_out[2 * b + 1] = (double)v[b].im; }
    }
    free(v);
  }
  if (!err) {
    R* tot = (R*)calloc(m, sizeof(R));
    for (uint64_t k = 0; k < na; k++)
      for (int i = 0; i < m; i++) {
        tot[i] += pa[k * m + i];
        if (per_a) per_a[k * m + i] = (double)pa[k * m + i];
      }
    for (int i = 0; i < m; i++) sums[i] = (double)tot[i];
    free(tot);
  }
  free(pa);
  return err;
}

/* ---------------------------------------------------------------------------------------------
 * finalize: Eq. (2) from the sums.
 *   alpha != 1 : M = log2(S_alpha / 2^N) / (1 - alpha)
 *   alpha == 1 : M_1 = -2^{-N} sum_P t log2 t     (q -> 1 limit, reading C4)
 *   lost_norm  = 1 - S_1 / 2^N
 * ------------------------------------------------------------------------------------------- */
int oracle_finalize(const double* sums, int N, const double* alpha, int n_alpha, double* M,
                    double* lost_norm) {
  const double D = ldexp(1.0, N);
  for (int i = 0; i < n_alpha; i++) {
    if (alpha[i] == 1.0)
      M[i] = -(sums[n_alpha + 1] / log(2.0)) / D;
    else
      M[i] = log2(sums[i] / D) / (1.0 - alpha[i]);
  }
  if (lost_norm) *lost_norm = 1.0 - sums[n_alpha] / D;
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* =============================================================================================
 * Qutrit mana (NEXT-3), Sec. 2.1 (Eqs. (4)-(10)) and Sec. 3.3 (Alg. 4, 5,
 * Eqs. (30)-(36)).  Index x = sum_j x_j 3^j (qutrit j is ternary digit j).
 * Each function returns sums[2] = { sum_u |<psi|A_u|psi>|, sum_u <psi|A_u|psi> } so that
 * mana = log2(sums[0] / 3^N) (Eq. (10)) and the Wigner normalisation sum_u W(u) = 1 reads
 * sums[1] = 3^N.
 * ============================================================================================= */
static uint64_t pow3(int n) { uint64_t r = 1; for (int i = 0; i < n; i++) r *= 3; return r; }
static int digit3(uint64_t x, int j) { for (int i = 0; i < j; i++) x /= 3; return (int)(x % 3); }
static uint64_t with_digit3(uint64_t x, int j, int d) {
  uint64_t p = pow3(j);
  return x - (uint64_t)digit3(x, j) * p + (uint64_t)d * p;
}
/* omega^k, omega = e^{2 pi i / 3} */
static C w3(int k) {
  k = ((k % 3) + 3) % 3;
  C c;
  c.re = cosl(2.0L * 3.14159265358979323846264338327950288L * k / 3.0L);
  c.im = sinl(2.0L * 3.14159265358979323846264338327950288L * k / 3.0L);
  return c;
}
static C cmul(C a, C b) { C c = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; return c; }

/* apply X^a (|k> -> |k+a>) or Z^b (|k> -> omega^{b k} |k>) to qutrit j of vector v (in place via tmp) */
static void q_apply_X(C* v, C* tmp, uint64_t D, int j, int a) {
  for (uint64_t x = 0; x < D; x++) tmp[with_digit3(x, j, (digit3(x, j) + a) % 3)] = v[x];
  memcpy(v, tmp, sizeof(C) * D);
}
static void q_apply_Z(C* v, uint64_t D, int j, int b) {
  for (uint64_t x = 0; x < D; x++) v[x] = cmul(w3(b * digit3(x, j)), v[x]);
}

/* Alg. 4 semantics: <psi| A_ab |psi> with A_ab = D A_0 D^dagger, D = prod_j X_j^{a_j} Z_j^{b_j}
 * (Eq. (30)) and A_0 |x> = |-x> (Eq. (31)), applied as operators: O(27^N). */
int oracle_mana_brute(const double* psi, int N, double* sums) {
  if (N < 1 || N > 6) return 1;
  const uint64_t D = pow3(N);
  R s_abs = 0.0L, s_sum = 0.0L;
  C* v = (C*)malloc(sizeof(C) * D);
  C* t = (C*)malloc(sizeof(C) * D);
  for (uint64_t a = 0; a < D; a++)
    for (uint64_t b = 0; b < D; b++) {
      for (uint64_t x = 0; x < D; x++) { v[x].re = psi[2 * x]; v[x].im = psi[2 * x + 1]; }
      /* D^dagger = (prod X^a Z^b)^dagger = prod Z^{-b} X^{-a} : apply X^{-a} first, then Z^{-b} */
      for (int j = 0; j < N; j++) q_apply_X(v, t, D, j, (3 - digit3(a, j)) % 3);
      for (int j = 0; j < N; j++) q_apply_Z(v, D, j, (3 - digit3(b, j)) % 3);
      for (uint64_t x = 0; x < D; x++) {                 /* A_0: |x> -> |-x> */
        uint64_t y = 0;
        for (int j = 0; j < N; j++) y += (uint64_t)((3 - digit3(x, j)) % 3) * pow3(j);
        t[y] = v[x];
      }
      memcpy(v, t, sizeof(C) * D);
      for (int j = 0; j < N; j++) q_apply_Z(v, D, j, digit3(b, j));   /* D = prod X^a Z^b: Z first */
      for (int j = 0; j < N; j++) q_apply_X(v, t, D, j, digit3(a, j));
      C e = {0.0L, 0.0L};
      for (uint64_t y = 0; y < D; y++) {
        R pr = psi[2 * y], pi = psi[2 * y + 1];
        e.re += pr * v[y].re + pi * v[y].im;
        e.im += pr * v[y].im - pi * v[y].re;
      }
      s_abs += sqrtl(e.re * e.re + e.im * e.im);
      s_sum += e.re;
    }
  free(v);
  free(t);
  sums[0] = (double)s_abs;
  sums[1] = (double)s_sum;
  return 0;
}

/* Phase-space definition, Eqs. (5)-(7): T_ab = omega^{-2^{-1} a b} Z^a X^b (2^{-1} = 2 mod 3),
 * T_u = (x)_j T_{u_j u'_j}, A_0 = 3^{-N} sum_u T_u, A_u = T_u A_0 T_u^dagger; returns sums of
 * <psi|A_u|psi> over all 9^N u.  Dense 3^N x 3^N matrices: N <= 3. */
int oracle_mana_phase_space(const double* psi, int N, double* sums) {
  if (N < 1 || N > 3) return 1;
  const uint64_t D = pow3(N), U = D * D;
  /* single-qutrit T_ab as 3x3 */
  C T1[9][3][3];
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++) {
      C ph = w3(-2 * a * b);
      for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) {
          /* (Z^a X^b)_{r c} = omega^{a r} [r == c + b] */
          C val = {0.0L, 0.0L};
          if (r == (c + b) % 3) val = cmul(ph, w3(a * r));
          T1[3 * a + b][r][c] = val;
        }
    }
  C* Tu = (C*)malloc(sizeof(C) * D * D);
  C* A0 = (C*)calloc(D * D, sizeof(C));
  C* Au = (C*)malloc(sizeof(C) * D * D);
  C* tmp = (C*)malloc(sizeof(C) * D * D);
  /* T_u element (r, c) = prod_j T1[u_j][r_j][c_j], u_j in 0..8 (digit pair) */
  for (uint64_t u = 0; u < U; u++) {
    for (uint64_t r = 0; r < D; r++)
      for (uint64_t c = 0; c < D; c++) {
        C v = {1.0L, 0.0L};
        uint64_t uu = u;
        for (int j = 0; j < N; j++) {
          int uj = (int)(uu % 9);
          uu /= 9;
          v = cmul(v, T1[uj][digit3(r, j)][digit3(c, j)]);
        }
        Tu[r * D + c] = v;
      }
    for (uint64_t k = 0; k < D * D; k++) { A0[k].re += Tu[k].re / (R)D; A0[k].im += Tu[k].im / (R)D; }
  }
  R s_abs = 0.0L, s_sum = 0.0L;
  for (uint64_t u = 0; u < U; u++) {
    for (uint64_t r = 0; r < D; r++)
      for (uint64_t c = 0; c < D; c++) {
        C v = {1.0L, 0.0L};
        uint64_t uu = u;
        for (int j = 0; j < N; j++) {
          int uj = (int)(uu % 9);
          uu /= 9;
          v = cmul(v, T1[uj][digit3(r, j)][digit3(c, j)]);
        }
        Tu[r * D + c] = v;
      }
    /* Au = Tu A0 Tu^dagger */
    for (uint64_t r = 0; r < D; r++)
      for (uint64_t c = 0; c < D; c++) {
        C acc = {0.0L, 0.0L};
        for (uint64_t k = 0; k < D; k++) { C p = cmul(Tu[r * D + k], A0[k * D + c]); acc.re += p.re; acc.im += p.im; }
        tmp[r * D + c] = acc;
      }
    for (uint64_t r = 0; r < D; r++)
      for (uint64_t c = 0; c < D; c++) {
        C acc = {0.0L, 0.0L};
        for (uint64_t k = 0; k < D; k++) {
          C td = {Tu[c * D + k].re, -Tu[c * D + k].im};     /* (Tu^dagger)_{k c} = conj(Tu_{c k}) */
          C p = cmul(tmp[r * D + k], td);
          acc.re += p.re;
          acc.im += p.im;
        }
        Au[r * D + c] = acc;
      }
    C e = {0.0L, 0.0L};                                     /* <psi|Au|psi> */
    for (uint64_t r = 0; r < D; r++)
      for (uint64_t c = 0; c < D; c++) {
        C pc = {psi[2 * c], psi[2 * c + 1]};
        C pr = {psi[2 * r], -psi[2 * r + 1]};
        C p = cmul(pr, cmul(Au[r * D + c], pc));
        e.re += p.re;
        e.im += p.im;
      }
    s_abs += sqrtl(e.re * e.re + e.im * e.im);
    s_sum += e.re;
  }
  free(Tu);
  free(A0);
  free(Au);
  free(tmp);
  sums[0] = (double)s_abs;
  sums[1] = (double)s_sum;
  return 0;
}

/* Alg. 5: for each a, alpha = X_a psi (alpha_x = psi_{x-a}), v_x = conj(alpha_x) alpha_{-x}
 * (Eq. (32)), chi = F_3^{(x)N} v with (F_3)_{jk} = omega^{2jk} (Eq. (35)), m += sum_b |chi_b|.
 * Naive radix-3 pass per digit.  a in [a_lo, a_hi); OpenMP over a. */
int oracle_mana_fwht(const double* psi, int N, uint64_t a_lo, uint64_t a_hi, double* sums) {
  if (N < 1 || N > 16 || a_lo > a_hi) return 1;
  const uint64_t D = pow3(N);
  if (a_hi > D) return 1;
  const uint64_t na = a_hi - a_lo;
  R* pa = (R*)calloc((size_t)(na ? na : 1) * 2, sizeof(R));
  uint64_t* p3 = (uint64_t*)malloc(sizeof(uint64_t) * (N + 1));
  for (int j = 0; j <= N; j++) p3[j] = pow3(j);
#pragma omp parallel
  {
    C* v = (C*)malloc(sizeof(C) * D);
    int* dg = (int*)malloc(sizeof(int) * N);
#pragma omp for schedule(dynamic, 1)
    for (int64_t k = 0; k < (int64_t)na; k++) {
      const uint64_t a = a_lo + (uint64_t)k;
      int ad[32];
      for (int j = 0; j < N; j++) ad[j] = (int)((a / p3[j]) % 3);
      for (uint64_t x = 0; x < D; x++) {
        uint64_t i1 = 0, i2 = 0;
        for (int j = 0; j < N; j++) {
          dg[j] = (int)((x / p3[j]) % 3);
          i1 += (uint64_t)((dg[j] - ad[j] + 3) % 3) * p3[j];         /* x - a      */
          i2 += (uint64_t)((6 - dg[j] - ad[j]) % 3) * p3[j];         /* (-x) - a   */
        }
        C al = {psi[2 * i1], psi[2 * i1 + 1]}, am = {psi[2 * i2], psi[2 * i2 + 1]};
        v[x].re = al.re * am.re + al.im * am.im;                     /* conj(alpha_x) alpha_{-x} */
        v[x].im = al.re * am.im - al.im * am.re;
      }
      C w[3] = {w3(0), w3(1), w3(2)};                                 /* omega^k, k mod 3 */
      for (int j = 0; j < N; j++) {                                   /* F_3 on digit j */
        const uint64_t h = p3[j];
        for (uint64_t base = 0; base < D; base += 3 * h)
          for (uint64_t o = 0; o < h; o++) {
            C u[3], y[3];
            for (int r = 0; r < 3; r++) u[r] = v[base + o + (uint64_t)r * h];
            for (int r = 0; r < 3; r++) {
              y[r].re = 0.0L; y[r].im = 0.0L;
              for (int c = 0; c < 3; c++) { C p = cmul(w[(2 * r * c) % 3], u[c]); y[r].re += p.re; y[r].im += p.im; }
            }
            for (int r = 0; r < 3; r++) v[base + o + (uint64_t)r * h] = y[r];
          }
      }
      R sa = 0.0L, ss = 0.0L;
      for (uint64_t b = 0; b < D; b++) { sa += sqrtl(v[b].re * v[b].re + v[b].im * v[b].im); ss += v[b].re; }
      pa[2 * k] = sa;
      pa[2 * k + 1] = ss;
    }
    free(v);
    free(dg);
  }
  R t0 = 0.0L, t1 = 0.0L;
  for (uint64_t k = 0; k < na; k++) { t0 += pa[2 * k]; t1 += pa[2 * k + 1]; }
  sums[0] = (double)t0;
  sums[1] = (double)t1;
  free(pa);
  free(p3);
  return 0;
}

/* =============================================================================================
 * Mixed-state qutrit mana (NEXT-4), Sec. 3.4 (Eq. (45), Alg. 6).
 * rho: 3^N x 3^N complex128, column-major (rho[r + c 3^N] = <r|rho|c>), as Alg. 6 requires.
 * sums[0] = sum_u |w_u|, sums[1] = sum_u Re w_u, w_u = Tr(rho A_u); mana = log2(sums[0] / 3^N)
 * (Eq. (10); reading C18 for the 1/3^N); sums[1] = 3^N Tr(rho).
 * ============================================================================================= */

/* single-qutrit A_u, u = 3a + b, as a 3x3 matrix: Eqs. (5)-(7) with N = 1, dense. */
static void qutrit_A1(C A[9][3][3]) {
  C T1[9][3][3];
  for (int a = 0; a < 3; a++)
    for (int b = 0; b < 3; b++) {
      C ph = w3(-2 * a * b);
      for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) {
          C val = {0.0L, 0.0L};
          if (r == (c + b) % 3) val = cmul(ph, w3(a * r));
          T1[3 * a + b][r][c] = val;
        }
    }
  C A0[3][3];
  memset(A0, 0, sizeof(A0));
  for (int u = 0; u < 9; u++)
    for (int r = 0; r < 3; r++)
      for (int c = 0; c < 3; c++) { A0[r][c].re += T1[u][r][c].re / 3.0L; A0[r][c].im += T1[u][r][c].im / 3.0L; }
  for (int u = 0; u < 9; u++) {
    C t[3][3];
    for (int r = 0; r < 3; r++)
      for (int c = 0; c < 3; c++) {
        C acc = {0.0L, 0.0L};
        for (int k = 0; k < 3; k++) { C p = cmul(T1[u][r][k], A0[k][c]); acc.re += p.re; acc.im += p.im; }
        t[r][c] = acc;
      }
    for (int r = 0; r < 3; r++)
      for (int c = 0; c < 3; c++) {
        C acc = {0.0L, 0.0L};
        for (int k = 0; k < 3; k++) {
          C td = {T1[u][c][k].re, -T1[u][c][k].im};
          C p = cmul(t[r][k], td);
          acc.re += p.re;
          acc.im += p.im;
        }
        A[u][r][c] = acc;
      }
  }
}

/* Phase-space definition for rho: w_u = Tr(rho A_u) with A_u = (x)_j A_{u_j} (Eqs. (5)-(7); the
 * N-qutrit A_u is the tensor product of single-qutrit ones because T_u and A_0 factorise).  Direct
 * O(9^N * 9^N) double sum: N <= 4. */
int oracle_mana_mixed_phase_space(const double* rho, int N, double* sums) {
  if (N < 1 || N > 4) return 1;
  const uint64_t D = pow3(N), U = D * D;
  C A1[9][3][3];
  qutrit_A1(A1);
  R s_abs = 0.0L, s_sum = 0.0L;
  for (uint64_t u = 0; u < U; u++) {
    C w = {0.0L, 0.0L};
    for (uint64_t r = 0; r < D; r++)
      for (uint64_t c = 0; c < D; c++) {
        /* Tr(rho A) = sum_{r,c} rho_{rc} A_{cr} */
        C a = {1.0L, 0.0L};
        uint64_t uu = u;
        for (int j = 0; j < N; j++) {
          a = cmul(a, A1[uu % 9][digit3(c, j)][digit3(r, j)]);
          uu /= 9;
        }
        C rv = {rho[2 * (r + c * D)], rho[2 * (r + c * D) + 1]};
        C p = cmul(rv, a);
        w.re += p.re;
        w.im += p.im;
      }
    s_abs += sqrtl(w.re * w.re + w.im * w.im);
    s_sum += w.re;
  }
  sums[0] = (double)s_abs;
  sums[1] = (double)s_sum;
  return 0;
}

/* Alg. 6 literally: M_{u,:} = vec(A_u^T)^T (column-major vec), Vec_N with
 * mu_k = 3 i_k + j_k and p = sum_k mu_k 9^{N-1-k} (i_k = ternary digit k of the row index r,
 * j_k of the column index c; reading C19), then the in-place leg sweep with the dense 9x9 M. */
int oracle_mana_mixed_alg6(const double* rho, int N, double* sums) {
  if (N < 1 || N > 8) return 1;
  const uint64_t D = pow3(N), V = D * D;
  C A1[9][3][3];
  qutrit_A1(A1);
  C M[9][9];
  for (int u = 0; u < 9; u++)
    for (int al = 0; al < 9; al++) {
      const int q = al % 3, p = al / 3;          /* column-major vec: alpha = q + 3p <-> (q, p) */
      M[u][al] = A1[u][p][q];                    /* (A_u^T)_{qp} = (A_u)_{pq} */
    }
  C* v = (C*)malloc(sizeof(C) * V);
  if (!v) return 2;
  for (uint64_t c = 0; c < D; c++)
    for (uint64_t r = 0; r < D; r++) {
      uint64_t p = 0;
      for (int k = 0; k < N; k++) p = 9 * p + (uint64_t)(3 * digit3(r, k) + digit3(c, k));
      v[p].re = rho[2 * (r + c * D)];
      v[p].im = rho[2 * (r + c * D) + 1];
    }
  for (int l = 0; l < N; l++) {
    uint64_t ns = 1;
    for (int k = 0; k < N - 1 - l; k++) ns *= 9;
    const uint64_t bs = 9 * ns, nb = V / bs;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < (int64_t)nb; b++)
      for (uint64_t m = 0; m < ns; m++) {
        const uint64_t base = (uint64_t)b * bs + m;
        C x[9], y[9];
        for (int a = 0; a < 9; a++) x[a] = v[base + (uint64_t)a * ns];
        for (int a = 0; a < 9; a++) {
          y[a].re = 0.0L;
          y[a].im = 0.0L;
          for (int k = 0; k < 9; k++) { C pr = cmul(M[a][k], x[k]); y[a].re += pr.re; y[a].im += pr.im; }
        }
        for (int a = 0; a < 9; a++) v[base + (uint64_t)a * ns] = y[a];
      }
  }
  R s_abs = 0.0L, s_sum = 0.0L;
  for (uint64_t k = 0; k < V; k++) { s_abs += sqrtl(v[k].re * v[k].re + v[k].im * v[k].im); s_sum += v[k].re; }
  free(v);
  sums[0] = (double)s_abs;
  sums[1] = (double)s_sum;
  return 0;
}
