/*
 * sre.h -- C ABI of libsre_b200.so: exact stabilizer Renyi entropy of N-qubit pure states on
 * NVIDIA B200 (sm_100a).
 *
 * Operation (PAPER.md = Sierant, Valles-Muns, Garcia-Saez, arXiv:2601.07824):
 *   M_alpha(|psi>) = 1/(1-alpha) log2[ sum_{a,b in Z_2^N} |<psi|X_a Z_b|psi>|^{2 alpha} / 2^N ]
 *       -- Eq. (2), with the modulus reading of chi^{2q} (reading C2);
 *   M_1 = -2^{-N} sum_P t log2 t, t = |<P>|^2  -- the alpha -> 1 limit (reading C4);
 *   lost_norm = 1 - sum_P <P>^2 / 2^N          -- P:1162.
 * computed by Algorithm 2: for every X-string a, chi_b(a) = sum_x conj(psi_{x^a}) psi_x
 * (-1)^{b.x} (Eq. (12)) for all b at once by a fast Walsh-Hadamard transform (Eq. (13)), and the
 * power sums of Eq. (11) accumulated in FP64.  The GPU kernels use the exact half-length
 * complex reformulation described in DESIGN.md ("Half-length transform").
 *
 * Conventions for every entry point:
 *   - psi: complex128 amplitudes, interleaved (re, im) doubles, index x = sum_j x_j 2^j (qubit j
 *     is bit j).  Batched calls take B contiguous states [B][2^N].  16-byte aligned.
 *   - Pointers are plain host or device addresses on the current CUDA device; no ownership is
 *     transferred; the library never frees caller memory.
 *   - Every function returns an int status (sre_status) and never aborts; on error the output
 *     buffers are left untouched and sre_last_error() holds a one-line reason.
 *   - Supported sizes: 1 <= N <= 26, 1 <= n_alpha <= 16, every alpha finite and > 0
 *     (alpha == 1 exactly selects the Shannon branch; reading C5).
 */
#ifndef SRE_B200_H
#define SRE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SRE_OK = 0,
  SRE_EINVAL = 1,      /* bad argument: null pointer, n_alpha out of range, alpha <= 0 / NaN */
  SRE_ERANGE = 2,      /* N outside [1, 26], B < 1, or a_begin/a_end outside [0, 2^N] */
  SRE_ENOTNORM = 3,    /* | ||psi||^2 - 1 | > 1e-8 (reading C6; checked by the synchronous calls) */
  SRE_EWORKSPACE = 4,  /* caller workspace smaller than sre_workspace_size() */
  SRE_ENOMEM = 5,      /* device allocation failed */
  SRE_ECUDA = 6,       /* CUDA runtime / launch error (text in sre_last_error) */
  SRE_EINTERNAL = 7,   /* internal consistency check failed */
  SRE_ENODEV = 8       /* no sm_100 device visible */
} sre_status;

#define SRE_MAX_N 26
#define SRE_MAX_ALPHA 16

/* Arithmetic of the transform (north star: FP64, with an optional FP32 mode).
 *   SRE_FP64: generation, Walsh-Hadamard transform, workspace and power sums in FP64
 *             (tolerance vs the oracle: S_alpha relative 1e-10).
 *   SRE_FP32: psi converted to complex64 once; generation, transform and workspace in FP32;
 *             each thread's 32-value tile summed in FP32, accumulated in FP64
 *             (tolerance: S_alpha relative 1e-4; halves the bytes moved per Pauli string). */
typedef enum { SRE_FP64 = 0, SRE_FP32 = 1 } sre_precision;

/* Static string for a status code. */
const char* sre_status_string(int code);
/* Thread-local detail of the last error (empty string if none). */
const char* sre_last_error(void);
/* ABI version (major*100 + minor). */
int sre_version(void);

/*
 * sre_exact -- M_alpha for one state, synchronous (Alg. 2 over all 2^N X-strings).
 *   psi      : host OR device pointer to 2^N complex128 (a host pointer is copied to the device
 *              inside the call: this is the end-to-end path).
 *   alpha    : host array [n_alpha] of Renyi indices.
 *   out_M    : host array [n_alpha], M_alpha in bits.
 *   out_lost_norm : host pointer to one double (nullable), lost_norm of P:1162.
 * Uses the legacy default stream and an internally cached workspace.
 */
int sre_exact(const void* psi, int N, const double* alpha, int n_alpha, double* out_M,
              double* out_lost_norm);

/*
 * sre_exact_batched -- B independent states psi[B][2^N] (BASELINE config 3).
 *   out_M : host [B][n_alpha] row-major; out_lost_norm : host [B] (nullable).
 */
int sre_exact_batched(const void* psi, int N, int B, const double* alpha, int n_alpha,
                      double* out_M, double* out_lost_norm);

/*
 * sre_workspace_size -- bytes of device workspace sre_partial_sums needs for (N, B, n_alpha).
 * Returns 0 for unsupported arguments.
 */
size_t sre_workspace_size(int N, int B, int n_alpha);

/*
 * sre_partial_sums -- asynchronous building block (multi-GPU sharding, checkpointed ranges).
 * Accumulates, for every state and for the X-strings a in [a_begin, a_end) only
 * (the chunked loop of P:314 / P:1179-1183), the raw sums of Eq. (11):
 *   sums_dev[s*(n_alpha+2) + i]         = sum_{a in range, b} t^{alpha_i}   (i < n_alpha)
 *   sums_dev[s*(n_alpha+2) + n_alpha]   = sum_{a in range, b} t             (purity, Eq. (14))
 *   sums_dev[s*(n_alpha+2) + n_alpha+1] = sum_{a in range, b} t ln t        (0 ln 0 = 0)
 * with t = |<psi|X_a Z_b|psi>|^2.  sums_dev is overwritten (device memory, [B][n_alpha+2]).
 * Sums over disjoint ranges add; they are deterministic for a given (range, N, B).
 *   psi       : device pointer, [B][2^N] complex128.
 *   alpha     : host array [n_alpha] (copied).
 *   workspace : device buffer of ws_bytes >= sre_workspace_size(N, B, n_alpha).
 *   stream    : cudaStream_t (NULL = legacy default stream); all work is enqueued on it.
 * No norm check (the caller owns it); a_begin == a_end writes zeros.
 */
int sre_partial_sums(const void* psi, int N, int B, uint64_t a_begin, uint64_t a_end,
                     const double* alpha, int n_alpha, void* workspace, size_t ws_bytes,
                     double* sums_dev, void* stream);

/*
 * sre_x_string_sums -- per-X-string sums for an arbitrary list of X-strings (NEXT-1 building block:
 * the "energy" of the thermodynamic-integration sampler, Eq. (17) f(X_a) = -ln S(a) with
 * S(a) = sum_b <psi|X_a Z_b|psi>^4, is one row of this output at alpha = 2; PAPER.md P:376-420,
 * Alg. 3 line "EvalEnergy").
 *   a_list : host array [n_a] of X-strings (each < 2^N), any order, repeats allowed.
 *   out_dev: device [n_a][n_alpha+2], row i = the sums of sre_partial_sums over [a_i, a_i + 1).
 *   workspace: >= sre_workspace_size(N, 1, n_alpha).  Enqueued on stream (async).
 */
int sre_x_string_sums(const void* psi, int N, const uint64_t* a_list, int n_a, const double* alpha, int n_alpha,
                      void* workspace, size_t ws_bytes, double* out_dev, void* stream);

/*
 * Precision-selecting variants (precision = sre_precision); the plain entry points are SRE_FP64.
 * sre_exact_ex takes B states like sre_exact_batched.  Unknown precision -> SRE_EINVAL (0 bytes
 * from sre_workspace_size_ex).
 */
size_t sre_workspace_size_ex(int N, int B, int n_alpha, int precision);
int sre_exact_ex(const void* psi, int N, int B, const double* alpha, int n_alpha, int precision, double* out_M,
                 double* out_lost_norm);
int sre_partial_sums_ex(const void* psi, int N, int B, uint64_t a_begin, uint64_t a_end, const double* alpha,
                        int n_alpha, int precision, void* workspace, size_t ws_bytes, double* sums_dev,
                        void* stream);

/*
 * sre_finalize -- host-side Eq. (2) from complete sums (all 2^N X-strings):
 *   alpha != 1: M = log2(S_alpha / 2^N) / (1 - alpha);  alpha == 1: M = -(sum t ln t)/(2^N ln 2);
 *   lost_norm = 1 - S_1 / 2^N.
 *   sums_host: [B][n_alpha+2] as produced by sre_partial_sums; out_M [B][n_alpha];
 *   out_lost_norm [B] (nullable).
 */
int sre_finalize(const double* sums_host, int N, int B, const double* alpha, int n_alpha,
                 double* out_M, double* out_lost_norm);

/*
 * sre_norm2 -- ||psi_s||^2 for each of B device states into device out_dev[B] (FP64, async).
 */
int sre_norm2(const void* psi, int N, int B, double* out_dev, void* stream);

/*
 * sre_chi -- debug/verification entry: chi_b(a) = <psi|X_a Z_b|psi> for one X-string a and all
 * b (Eq. (12)), computed by the kernels that evaluate that X-string in the sums -- the single-pass
 * kernels for N <= 14; for N >= 15 the production staged (N <= 20) or streamed (N = 21..24) pass A
 * and TMA pass B when a >= 2^L and a % 8 == 0 (their pass-B epilogue decodes every output), else
 * the generic two-pass kernels that take such head X-strings in the sums -- written to device
 * chi_dev[2*2^N] as complex128 in natural b order (each chi is purely real or purely imaginary,
 * DESIGN C3).  Synchronous on `stream`.
 */
int sre_chi(const void* psi, int N, uint64_t a, double* chi_dev, void* stream);

/*
 * sre_pauli_spectrum -- spectrum epilogue (NEXT-2): histogram of t = |<psi|P|psi>|^2 over the
 * Pauli strings of the X-strings a in [a_begin, a_end) (all 2^N Z-strings of each), from the same
 * kernels as the sums (single-pass for N <= 14, pass-B epilogues for N >= 15).  Bin k (k <= 62)
 * counts round(-log2 t) == k, i.e. t in (2^{-k-1/2}, 2^{-k+1/2}]; bin 63 counts t < 2^{-62.5}
 * and exact zeros (DESIGN C22).
 *   hist_dev : device uint64[64], overwritten.
 *   workspace >= sre_workspace_size(N, 1, 1) + 256 (the tail holds scratch sums for N >= 15).
 * Errors: SRE_ERANGE (bad range), SRE_EINVAL (also: opt-in SRE_FUSED / SRE_TMEM kernels set),
 * SRE_EWORKSPACE, SRE_ECUDA.  Enqueued on stream; integer counts, exact and order-independent.
 */
int sre_pauli_spectrum(const void* psi, int N, uint64_t a_begin, uint64_t a_end, uint64_t* hist_dev, void* workspace,
                       size_t ws_bytes, void* stream);

/*
 * Instrumentation used by bench.py (no effect on results).
 *   sre_launch_count   : cumulative number of kernels this library launched in the process.
 *   sre_profile_begin  : start sampling; every stride-th launch of each kernel kind is bracketed
 *                        by CUDA events on its own stream.
 *   sre_profile_end    : stop; per kind k (0 single-pass, 1 pass A, 2 pass B, 3 auxiliary,
 *                        4 fused persistent two-pass)
 *                        ms_sum[k] = summed event time of the sampled launches, n_timed[k] = how
 *                        many were sampled, n_launched[k] = launches of that kind since begin.
 *                        Arrays have 5 entries each (any may be NULL).  Synchronises the events.
 */
uint64_t sre_launch_count(void);
int sre_profile_begin(int stride);
int sre_profile_end(double* ms_sum, uint64_t* n_timed, uint64_t* n_launched);

/* ============================================================================================
 * Pure-state qutrit mana (NEXT-3): Algorithm 5, Sec. 3.3.2.
 *
 * psi: 3^N complex128 amplitudes (interleaved re, im; 16-byte aligned), index x = sum_j x_j 3^j
 * (qutrit j = ternary digit j; DESIGN C19).  For each X-string a in Z_3^N the library forms
 * v_x = conj(psi_{x-a}) psi_{-x-a} (Eq. (32), digit-wise mod 3), chi(a) = F_3^{(x)N} v with
 * (F_3)_{jk} = omega^{2jk}, omega = e^{2 pi i/3} (Eqs. (35)-(36)), and accumulates in FP64
 *   S_abs = sum_{a,b} |chi_b(a)|      S_sum = sum_{a,b} chi_b(a)  ( = 3^N ||psi||^2 ).
 * Mana = log2(S_abs / 3^N) (Eq. (10) / (11), DESIGN C18).  N in [1, SRE_MANA_MAX_N].
 * ============================================================================================ */
#define SRE_MANA_MAX_N 16

/* Bytes of device workspace sre_mana_partial_sums prefers for N (0 if N is out of range): about
 * 2 GiB of X-string pairs per launch for N >= 9 (64 KiB for N <= 8).  Less is accepted down to
 * the size of one X-string pair; fewer pairs then run per launch (slower; equal up to FP64
 * reassociation). */
size_t sre_mana_workspace_size(int N);

/*
 * sre_mana_partial_sums -- asynchronous building block (multi-GPU shards, checkpointed ranges).
 *   psi       : DEVICE pointer to 3^N complex128 (not modified; not checked for normalisation).
 *   [a_begin, a_end) : X-string range, 0 <= a_begin <= a_end <= 3^N (X-string a as a base-3 integer).
 *   workspace : device buffer, 256-byte aligned, ws_bytes bytes (>= one pair; see above).
 *   sums_dev  : device double[2] <- (S_abs, S_sum) restricted to the range (overwritten).
 *   stream    : cudaStream_t (NULL = legacy default stream).  Enqueues only; no host sync.
 * Errors: SRE_EINVAL (NULL / misaligned / host psi), SRE_ERANGE (N or range), SRE_EWORKSPACE,
 * SRE_ECUDA.  Deterministic: bitwise identical results for the same inputs on the same device.
 */
int sre_mana_partial_sums(const void* psi, int N, uint64_t a_begin, uint64_t a_end, void* workspace,
                          size_t ws_bytes, double* sums_dev, void* stream);

/*
 * sre_mana -- synchronous convenience: mana of one state, psi a HOST or DEVICE pointer.
 *   out_mana  : log2(S_abs / 3^N).   out_norm2 (may be NULL): S_sum / 3^N = ||psi||^2.
 * Returns SRE_ENOTNORM (with out_norm2 set, out_mana untouched) when | ||psi||^2 - 1 | > 1e-8.
 * Uses library-owned cached device buffers (one per process, guarded by a mutex).
 */
int sre_mana(const void* psi, int N, double* out_mana, double* out_norm2);

/*
 * sre_mana_finalize -- host-side Eq. (10) (DESIGN C18) from complete sums over
 * all 3^N X-strings (e.g. sre_mana_partial_sums shards added over ranks):
 *   sums_host : HOST double[2] = (S_abs, S_sum).
 *   out_mana  : log2(S_abs / 3^N).   out_norm2 (may be NULL): S_sum / 3^N = ||psi||^2.
 * Errors: SRE_EINVAL (NULL, S_abs <= 0), SRE_ERANGE (N).  No device work; needs no GPU.
 */
int sre_mana_finalize(const double* sums_host, int N, double* out_mana, double* out_norm2);

/* ============================================================================================
 * Mixed-state qutrit mana (NEXT-4): Algorithm 6, Sec. 3.4 (Eq. (45)).
 *
 * rho: 3^N x 3^N complex128, COLUMN-MAJOR (rho[r + c 3^N] = <r|rho|c>, Alg. 6's input), 16-byte
 * aligned; qutrit j = ternary digit j of r and c (DESIGN C19).  The library applies M^{(x)N}
 * (w_u = Tr(rho A_u)) leg by leg and accumulates in FP64
 *   S_abs = sum_u |w_u|      S_sum = sum_u w_u  ( = 3^N Tr rho ).
 * Mana = log2(S_abs / 3^N) (Eq. (10), DESIGN C18/C20).  N in [1, SRE_MANA_MIXED_MAX_N]
 * (N = 10 is 9^10 x 16 B = 56 GB of HBM).
 * ============================================================================================ */
#define SRE_MANA_MIXED_MAX_N 10

/* Bytes of device workspace sre_mana_mixed_sums needs (per-CTA accumulator slots). */
size_t sre_mana_mixed_workspace_size(int N);

/*
 * sre_mana_mixed_sums -- asynchronous, IN PLACE: rho (DEVICE pointer) is overwritten by w
 * (transformed through all but the last leg; its contents are unspecified afterwards).
 *   sums_dev : device double[2] <- (S_abs, S_sum).   stream: cudaStream_t (NULL = default).
 * Errors: SRE_EINVAL (NULL / misaligned / host rho), SRE_ERANGE (N), SRE_EWORKSPACE, SRE_ECUDA.
 */
int sre_mana_mixed_sums(void* rho, int N, void* workspace, size_t ws_bytes, double* sums_dev, void* stream);

/*
 * sre_mana_mixed -- synchronous convenience; rho is a HOST or DEVICE pointer and is not modified
 * (copied into a library-owned device buffer of 9^N x 16 bytes).
 *   out_mana : log2(S_abs / 3^N).   out_trace (may be NULL): S_sum / 3^N = Tr rho.
 * Returns SRE_ENOTNORM (out_trace set, out_mana untouched) when |Tr rho - 1| > 1e-8.
 */
int sre_mana_mixed(const void* rho, int N, double* out_mana, double* out_trace);

#ifdef __cplusplus
}
#endif

#endif /* SRE_B200_H */
