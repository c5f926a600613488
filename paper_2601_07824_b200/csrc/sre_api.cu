// sre_api.cu -- C ABI of libsre_b200.so (include/sre.h): validation, planning, workspace,
// launch schedule and finalisation for the exact SRE hot path (Alg. 2).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <type_traits>
#include <vector>

#include "../../include/sre.h"
#define SRE_API_TU
#include "launch.cuh"

using namespace sre;
using namespace sre_host;

namespace sre_host {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) return fail(SRE_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                   \
  } while (0)

// ------------------------------------------------------------------------------------------
// launch accounting and sampled per-kernel timing (bench.py's roofline numbers)
// ------------------------------------------------------------------------------------------
Prof g_prof;
std::atomic<uint64_t> g_launches{0};

cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) {
    cudaEvent_t e = g_prof.pool.back();
    g_prof.pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}


int get_dev(Dev& d) {
  int id = 0;
  cudaError_t e = cudaGetDevice(&id);
  if (e != cudaSuccess) return fail(SRE_ENODEV, "cudaGetDevice: %s", cudaGetErrorString(e));
  static std::mutex mu;
  static Dev cache[64];
  std::lock_guard<std::mutex> lk(mu);
  if (id < 0 || id >= 64) return fail(SRE_ENODEV, "device id %d", id);
  if (cache[id].id != id) {
    cudaDeviceProp pr;
    CK(cudaGetDeviceProperties(&pr, id));
    if (pr.major != 10) return fail(SRE_ENODEV, "device %d is sm_%d%d; libsre_b200 is built for sm_100a", id, pr.major, pr.minor);
    cache[id].id = id;
    cache[id].sms = pr.multiProcessorCount;
    cache[id].major = pr.major;
    cache[id].minor = pr.minor;
  }
  d = cache[id];
  return SRE_OK;
}

// ------------------------------------------------------------------------------------------
// plan
// ------------------------------------------------------------------------------------------
int staged_groups(int N) {
  const char* e = getenv("SRE_KG");
  if (e && atoi(e) > 0) return atoi(e) > 1024 ? 1024 : atoi(e);
  // 8-X-string groups per staged launch pair, measured on B200: launch tails
  // dominate small batches (N = 20 with 8 X-strings per launch pair: 6.3 us per X-string, L2-resident
  // workspace or not), so N <= 18 takes 4096 X-strings per launch (<= 8 GiB of workspace);
  // N = 19 saturates at 512.
  if (N <= 18) return 512;
  if (N == 19) return 64;
  return 32;   // N = 20: 256 X-strings (2 GiB) per launch pair, measured 3.47 vs 3.57 us per X-string at 128 (r02)
}

void two_pass_params(int T, int& L, int& H, int& CB) {
  L = T - 9;
  if (L < 10) L = 10;
  if (L > 13) L = 13;
  if (T >= 20 && T <= 23) L = 12;   // streamed path (N = 21..24): two 128-thread units per CTA
  if (T == 24) L = 13;              // N = 25: one 256-thread unit (keeps pass-B rows >= 32 B)
  H = T - L;
  CB = 13 - H;
  if (CB > 6) CB = 6;
  if (CB < 2) CB = 2;
}

constexpr int SMALL_MAX_T = 10;
constexpr int MID_MAX_T = 13;

// CTAs per state for the single-pass kernels: minimise waves x per-CTA items (uniform cost).  With
// slack > 0 the smallest g within (1 + slack) of that minimum: fewer, longer CTAs amortise a per-CTA
// start (k_midr's ring fill) at no modelled cost.
int pick_gx(uint64_t count, int per_cta, int B, int resident, double slack = 0.0) {
  const uint64_t maxg = (count + per_cta - 1) / per_cta;
  auto cost = [&](int g) {
    const uint64_t waves = ((uint64_t)B * g + resident - 1) / resident;
    const uint64_t items = (count + (uint64_t)g * per_cta - 1) / ((uint64_t)g * per_cta);
    return waves * items;
  };
  uint64_t best = ~0ull;
  int bg = 1;
  for (int g = 1; g <= 4096 && (uint64_t)g <= maxg; ++g)
    if (cost(g) < best) { best = cost(g); bg = g; }
  if (slack > 0.0)
    for (int g = 1; g < bg; ++g)
      if ((double)cost(g) <= (double)best * (1.0 + slack)) return g;
  return bg;
}

// count: X-strings the call will evaluate (the staged batch never exceeds it, so short ranges and
// single X-strings -- sre_x_string_sums, sre_chi, Monte-Carlo energies -- keep small slot arrays).
int make_plan(int N, const Dev& d, Plan& p, uint64_t count = ~0ull) {
  p.N = N;
  p.T = N - 1;
  if (p.T <= SMALL_MAX_T) {
    p.kind = SMALL;
    p.slots = 4096;
  } else if (p.T <= MID_MAX_T) {
    p.kind = MID;
    p.slots = 4096;
  } else {
    p.kind = TWOPASS;
    two_pass_params(p.T, p.L, p.H, p.CB);
    p.TP = p.CB + p.H;
    uint64_t k = (1ull << 23) >> N;  // K * 2^N doubles ~ 64 MiB of workspace in flight
    if (k < 8) k = 8;                 // N >= 21: HBM workspace; 8 X-strings share each psi row pair
    if (k > 64) k = 64;
    p.K = (int)k;
    p.unitsA = 256 >> (p.L - 5);
    p.blkB = p.TP >= 14 ? 512 : 256;
    p.unitsB = p.blkB >> (p.TP - 5);
    p.slab_doubles = (size_t)p.K << N;
    const uint64_t itemsB = (uint64_t)p.K * 2 * (1ull << (p.L - p.CB));
    p.slots = (size_t)((itemsB + p.unitsB - 1) / p.unitsB);
    if (N >= 21 && N <= 25) {  // streamed pass A (k_passAr / k_passAs) + TMA-fed pass B with 2^13-double tiles
      // X-strings per launch pair: the launch's groups read each psi row pair from L2 after its first
      // HBM fetch, so psi traffic per X-string is 2^(N+4) / K bytes (N = 24, K = 32: 8 MiB vs a
      // 128 MiB workspace round trip); workspace K x 2^(N+3) bytes (N = 24: 4 GiB)
      int kk = N == 21 ? 64 : 32;
      if (const char* e = getenv("SRE_K")) {   // experiments: X-strings per streamed launch pair
        const int ke = atoi(e);
        if (ke >= 8 && ke <= 512) kk = ke & ~7;
      }
      if ((uint64_t)kk > count) kk = (int)(((count + 7) / 8) * 8 > 0 ? ((count + 7) / 8) * 8 : 8);
      p.K = kk;
      p.KG = kk / 8;
      p.slab_doubles = (size_t)p.K << N;
      p.slots = (size_t)(((uint64_t)p.K * 2 * (1ull << (p.L - p.CB)) + p.unitsB - 1) / p.unitsB);
      p.staged = true;
      p.amin = 1ull << p.L;
      if (p.slots < 4 * 160) p.slots = 4 * 160;
    }
    if (p.L == 10) {  // staged pass A + persistent pass B (N = 15..20)
      p.staged = true;
      p.KG = staged_groups(N);
      if ((uint64_t)8 * p.KG > count) p.KG = (int)((count + 7) / 8 > 0 ? (count + 7) / 8 : 1);
      if ((size_t)8 * p.KG > (size_t)p.K) {
        p.K = 8 * p.KG;
        p.slab_doubles = (size_t)p.K << N;
        const uint64_t itemsK = (uint64_t)p.K * 2 * (1ull << (p.L - p.CB));  // generic pass B grid for K
        p.slots = (size_t)((itemsK + p.unitsB - 1) / p.unitsB);
      }
      if (p.slots < 4 * 160) p.slots = 4 * 160;  // persistent grids: <= 4 CTAs x SMs
      p.amin = 1024;
    }
  }
  (void)d;
  return SRE_OK;
}

// Workspace layout (bytes, every region 256-B aligned for bulk copies):
//   [partial slots][slab][norm scratch][Ctl][psi as complex64 (FP32 mode only)]
constexpr size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }
size_t off_slab(const Plan& p, int B) { return align256(p.slots * NACC * (p.kind == TWOPASS ? 1 : (size_t)B) * 8); }
size_t off_norm(const Plan& p, int B) { return off_slab(p, B) + align256(p.slab_doubles * 8); }
size_t off_ctl(const Plan& p, int B) { return off_norm(p, B) + align256((4096 * (size_t)B + (size_t)B) * 8); }
size_t off_psi32(const Plan& p, int B) { return off_ctl(p, B) + align256(sizeof(Ctl)); }
size_t ws_bytes_for(const Plan& p, int B, int prec = 0) {
  return off_psi32(p, B) + (prec ? align256(((size_t)B << p.N) * sizeof(float2)) : 0);
}
Ctl* ctl_of(char* ws, const Plan& p, int B) { return reinterpret_cast<Ctl*>(ws + off_ctl(p, B)); }
float2* psi32_of(char* ws, const Plan& p, int B) { return reinterpret_cast<float2*>(ws + off_psi32(p, B)); }

// ------------------------------------------------------------------------------------------
// alpha sweeps
// ------------------------------------------------------------------------------------------
struct Sweep {
  Alphas al;
  int first = 0;
  bool a2 = false;
  double scale4[MAXA];
};

std::vector<Sweep> make_sweeps(const double* alpha, int n_alpha) {
  std::vector<Sweep> sw;
  bool any_one = false;
  for (int i = 0; i < n_alpha; ++i) any_one |= (alpha[i] == 1.0);
  for (int f = 0; f < n_alpha; f += MAXA) {
    Sweep s;
    memset(&s.al, 0, sizeof(s.al));
    s.first = f;
    s.al.n = n_alpha - f < MAXA ? n_alpha - f : MAXA;
    s.al.need_log = (f == 0 && any_one) ? 1 : 0;
    for (int i = 0; i < s.al.n; ++i) {
      const double a = alpha[f + i];
      s.al.alpha[i] = a;
      if (a == std::floor(a) && a >= 1.0 && a <= 64.0) {
        s.al.kind[i] = 0;
        s.al.iexp[i] = (int)a;
      } else {
        s.al.kind[i] = 2;
        s.al.iexp[i] = 0;
        s.al.any_real = 1;
      }
      s.scale4[i] = std::pow(4.0, a);  // t = 4 t'  =>  t^alpha = 4^alpha t'^alpha
    }
    s.a2 = (s.al.n == 1 && alpha[f] == 2.0 && !s.al.need_log);
    sw.push_back(s);
  }
  return sw;
}

int occupancy_small(int T, const Dev& d) {
  (void)T;
  return 4 * d.sms;  // 256-thread CTAs, modest registers
}

// ------------------------------------------------------------------------------------------
// the range driver: sums_dev[B][n_alpha+2] for a in [a_begin, a_end)
// ------------------------------------------------------------------------------------------
// V = double: FP64 path; V = float: FP32 mode (psi already converted to complex64)
template <class V>
int run_range_t(const typename Cx<V>::T* psi, const Plan& p, const Dev& d, int N, int B, uint64_t a_begin,
                uint64_t a_end, const double* alpha, int n_alpha, char* ws, double* sums_dev, cudaStream_t st,
                unsigned long long* hist = nullptr) {
  double* partial = reinterpret_cast<double*>(ws);
  V* slab = reinterpret_cast<V*>(ws + off_slab(p, B));
  Ctl* ctl = ctl_of(ws, p, B);
  CK(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
  const uint64_t count = a_end - a_begin;
  CK(cudaMemsetAsync(sums_dev, 0, sizeof(double) * (size_t)B * (n_alpha + 2), st));
  if (count == 0) return SRE_OK;
  const std::vector<Sweep> sweeps = make_sweeps(alpha, n_alpha);
  for (const Sweep& sw : sweeps) {
    Alphas al_h = sw.al;   // spectrum epilogue pointer rides in the alphas (two-pass kernels)
    al_h.hist = hist;
    ReduceArgs ra;
    memset(&ra, 0, sizeof(ra));
    ra.n_alpha = n_alpha;
    ra.first = sw.first;
    ra.n_this = sw.al.n;
    ra.write_common = sw.first == 0;
    for (int i = 0; i < MAXA; ++i) ra.scale4[i] = sw.scale4[i];
    ra.err = &ctl->error;
    if (p.kind == SMALL || p.kind == MID) {
      int gx;
      if (p.kind == SMALL) {
        const int G = p.T >= 5 ? 32 : (1 << p.T);
        gx = pick_gx(count, 256 / G, B, occupancy_small(p.T, d));
      } else {
        gx = pick_gx(count, 256 >> (p.T - 5), B, d.sms, 0.01);
      }
      if ((size_t)gx > p.slots) gx = (int)p.slots;
      CK(cudaMemsetAsync(partial, 0, sizeof(double) * (size_t)gx * B * NACC, st));
      cudaError_t e;
      if (p.kind == SMALL)
        e = sw.a2 ? launch_small<V, true, false>(p.T, psi, N, B, gx, a_begin, count, al_h, partial, nullptr, st, nullptr)
                  : launch_small<V, false, false>(p.T, psi, N, B, gx, a_begin, count, al_h, partial, nullptr, st, nullptr);
      else
        e = sw.a2 ? launch_mid<V, true, false>(p.T, psi, N, B, gx, a_begin, count, al_h, partial, nullptr, st, nullptr)
                  : launch_mid<V, false, false>(p.T, psi, N, B, gx, a_begin, count, al_h, partial, nullptr, st, nullptr);
      if (e != cudaSuccess) return fail(SRE_ECUDA, "launch: %s", cudaGetErrorString(e));
      ra.nslots = gx;
      CK(launch_counted(LK_AUX, st, [&] { k_reduce<<<B, 256, 0, st>>>(partial, ra, sums_dev); return cudaGetLastError(); }));
    } else {
      for (int s = 0; s < B; ++s) {
        const typename Cx<V>::T* ps = psi + ((size_t)s << N);
        CK(cudaMemsetAsync(partial, 0, sizeof(double) * p.slots * NACC, st));
        // generic batches (a < 2^L, unaligned heads, L > 10): k_passA + k_passB
        auto generic = [&](uint64_t lo, uint64_t hi) -> int {
          for (uint64_t a = lo; a < hi; a += (uint64_t)p.K) {
            const int kc = (int)((hi - a) < (uint64_t)p.K ? (hi - a) : (uint64_t)p.K);
            cudaError_t e = launch_passA<V>(p, ps, a, kc, slab, st);
            if (e != cudaSuccess) return fail(SRE_ECUDA, "passA: %s", cudaGetErrorString(e));
            e = sw.a2 ? launch_passB<V, true, false>(p, a, kc, slab, al_h, partial, nullptr, st)
                      : launch_passB<V, false, false>(p, a, kc, slab, al_h, partial, nullptr, st);
            if (e != cudaSuccess) return fail(SRE_ECUDA, "passB: %s", cudaGetErrorString(e));
          }
          return SRE_OK;
        };
        if (!p.staged) {
          int rc2 = generic(a_begin, a_end);
          if (rc2) return rc2;
        } else {
          // staged groups need 8-aligned X-strings with a_h = a >> L != 0
          uint64_t s0 = a_begin < p.amin ? p.amin : a_begin;
          s0 = (s0 + 7) & ~7ull;
          if (s0 > a_end) s0 = a_end;
          int rc2 = generic(a_begin, s0);
          if (rc2) return rc2;
          const uint64_t per = (uint64_t)8 * p.KG;
          for (uint64_t a = s0; a < a_end; a += per) {
            const int kc = (int)((a_end - a) < per ? (a_end - a) : per);
            cudaError_t e = launch_passA10s<V>(p, d, ps, a, kc, slab, st);
            if (e != cudaSuccess) return fail(SRE_ECUDA, "passA10s: %s", cudaGetErrorString(e));
            e = sw.a2 ? launch_passBp<V, true>(p, d, kc, slab, al_h, partial, st)
                      : launch_passBp<V, false>(p, d, kc, slab, al_h, partial, st);
            if (e != cudaSuccess) return fail(SRE_ECUDA, "passBp: %s", cudaGetErrorString(e));
          }
        }
        ra.nslots = (int)p.slots;
        CK(launch_counted(LK_AUX, st, [&] {
          k_reduce<<<1, 256, 0, st>>>(partial, ra, sums_dev + (size_t)s * (n_alpha + 2));
          return cudaGetLastError();
        }));
      }
    }
  }
  return SRE_OK;
}

int run_range(const double2* psi, int N, int B, uint64_t a_begin, uint64_t a_end, const double* alpha, int n_alpha,
              char* ws, size_t ws_bytes, double* sums_dev, cudaStream_t st, int prec = SRE_FP64,
              unsigned long long* hist = nullptr) {
  Dev d;
  int rc = get_dev(d);
  if (rc) return rc;
  Plan p;
  make_plan(N, d, p, a_end - a_begin);
  if (ws_bytes < ws_bytes_for(p, B, prec))
    return fail(SRE_EWORKSPACE, "workspace %zu < required %zu", ws_bytes, ws_bytes_for(p, B, prec));
  if (prec == SRE_FP32) {
    float2* p32 = psi32_of(ws, p, B);
    const uint64_t n = (uint64_t)B << N;
    CK(launch_counted(LK_AUX, st, [&] { k_to_f32<<<4 * d.sms, 256, 0, st>>>(psi, p32, n); return cudaGetLastError(); }));
    return run_range_t<float>(p32, p, d, N, B, a_begin, a_end, alpha, n_alpha, ws, sums_dev, st);
  }
  return run_range_t<double>(psi, p, d, N, B, a_begin, a_end, alpha, n_alpha, ws, sums_dev, st, hist);
}

int validate_common(const void* psi, int N, int B, const double* alpha, int n_alpha) {
  if (!psi) return fail(SRE_EINVAL, "psi is NULL");
  if (N < 1 || N > SRE_MAX_N) return fail(SRE_ERANGE, "N=%d outside [1, %d]", N, SRE_MAX_N);
  if (B < 1) return fail(SRE_ERANGE, "B=%d < 1", B);
  if (!alpha) return fail(SRE_EINVAL, "alpha is NULL");
  if (n_alpha < 1 || n_alpha > SRE_MAX_ALPHA) return fail(SRE_EINVAL, "n_alpha=%d outside [1, %d]", n_alpha, SRE_MAX_ALPHA);
  for (int i = 0; i < n_alpha; ++i)
    if (!(alpha[i] > 0.0) || !std::isfinite(alpha[i])) return fail(SRE_EINVAL, "alpha[%d]=%g must be finite and > 0", i, alpha[i]);
  if (reinterpret_cast<uintptr_t>(psi) % 16) return fail(SRE_EINVAL, "psi not 16-byte aligned");
  return SRE_OK;
}

int is_device_ptr(const void* ptr, bool& dev) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    dev = false;
    return SRE_OK;
  }
  dev = (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
  return SRE_OK;
}

// List mode (sre_x_string_sums, N <= 14): one launch per alpha sweep evaluates every X-string of
// alist_dev (device, n_a <= kListMax); item i's sums land in partial[i] and k_reduce (one block
// per item, one slot each) writes out_dev row i.  Replaces n_a range calls (5 launches each).
constexpr int kListMax = 2048;

int run_list(const double2* psi, int N, const uint64_t* alist_dev, int n_a, const double* alpha, int n_alpha,
             char* ws, double* out_dev, cudaStream_t st) {
  Dev d;
  int rc = get_dev(d);
  if (rc) return rc;
  Plan p;
  make_plan(N, d, p, 1);
  if (!(p.kind == SMALL || p.kind == MID)) return fail(SRE_EINTERNAL, "list mode needs N <= 14");
  double* partial = reinterpret_cast<double*>(ws);
  const std::vector<Sweep> sweeps = make_sweeps(alpha, n_alpha);
  for (const Sweep& sw : sweeps) {
    ReduceArgs ra;
    memset(&ra, 0, sizeof(ra));
    ra.n_alpha = n_alpha;
    ra.first = sw.first;
    ra.n_this = sw.al.n;
    ra.write_common = sw.first == 0;
    for (int i = 0; i < MAXA; ++i) ra.scale4[i] = sw.scale4[i];
    ra.err = nullptr;
    ra.nslots = 1;
    int gx;
    cudaError_t e;
    if (p.kind == SMALL) {
      const int G = p.T >= 5 ? 32 : (1 << p.T);
      gx = pick_gx(n_a, 256 / G, 1, occupancy_small(p.T, d));
      e = sw.a2 ? launch_small<double, true, false>(p.T, psi, N, 1, gx, 0, n_a, sw.al, partial, nullptr, st, alist_dev)
                : launch_small<double, false, false>(p.T, psi, N, 1, gx, 0, n_a, sw.al, partial, nullptr, st, alist_dev);
    } else {
      gx = pick_gx(n_a, 256 >> (p.T - 5), 1, d.sms);
      e = sw.a2 ? launch_mid<double, true, false>(p.T, psi, N, 1, gx, 0, n_a, sw.al, partial, nullptr, st, alist_dev)
                : launch_mid<double, false, false>(p.T, psi, N, 1, gx, 0, n_a, sw.al, partial, nullptr, st, alist_dev);
    }
    if (e != cudaSuccess) return fail(SRE_ECUDA, "list launch: %s", cudaGetErrorString(e));
    CK(launch_counted(LK_AUX, st, [&] { k_reduce<<<n_a, 256, 0, st>>>(partial, ra, out_dev); return cudaGetLastError(); }));
  }
  return SRE_OK;
}

// internal cached device buffers for the synchronous calls
struct Cache {                 // one per device: buffers stay with the device that allocated them
  char* ws = nullptr;
  size_t ws_bytes = 0;
  char* in = nullptr;
  size_t in_bytes = 0;
};
std::mutex g_cache_mu;
Cache g_caches[64];

int cache_get(char** buf, size_t* have, size_t need) {
  if (*have >= need) return SRE_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *have = 0;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(buf), need);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SRE_ENOMEM, "cudaMalloc(%zu): %s", need, cudaGetErrorString(e));
  }
  *have = need;
  return SRE_OK;
}

int exact_impl(const void* psi, int N, int B, const double* alpha, int n_alpha, double* out_M, double* out_ln,
               int prec = SRE_FP64) {
  if (prec != SRE_FP64 && prec != SRE_FP32) return fail(SRE_EINVAL, "precision %d", prec);
  int rc = validate_common(psi, N, B, alpha, n_alpha);
  if (rc) return rc;
  if (!out_M) return fail(SRE_EINVAL, "out_M is NULL");
  Dev d;
  rc = get_dev(d);
  if (rc) return rc;
  bool dev_ptr = false;
  is_device_ptr(psi, dev_ptr);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  Cache& g_cache = g_caches[d.id];
  Plan p;
  make_plan(N, d, p);
  const size_t need = ws_bytes_for(p, B, prec) + sizeof(double) * ((size_t)B * (n_alpha + 2) + (size_t)B);
  rc = cache_get(&g_cache.ws, &g_cache.ws_bytes, need);
  if (rc) return rc;
  cudaStream_t st = 0;
  const double2* dpsi = reinterpret_cast<const double2*>(psi);
  const size_t psi_bytes = ((size_t)B << N) * sizeof(double2);
  if (!dev_ptr) {
    rc = cache_get(&g_cache.in, &g_cache.in_bytes, psi_bytes);
    if (rc) return rc;
    CK(cudaMemcpyAsync(g_cache.in, psi, psi_bytes, cudaMemcpyHostToDevice, st));
    dpsi = reinterpret_cast<const double2*>(g_cache.in);
  }
  double* sums = reinterpret_cast<double*>(g_cache.ws + ws_bytes_for(p, B, prec));
  double* norms = sums + (size_t)B * (n_alpha + 2);
  // norm check (reading C6)
  {
    double* part = reinterpret_cast<double*>(g_cache.ws + off_norm(p, B));  // the norm area
    const int nb = 64;
    dim3 g(nb, B);
    CK(launch_counted(LK_AUX, st, [&] { k_norm2_partial<<<g, 256, 0, st>>>(dpsi, N, part); return cudaGetLastError(); }));
    CK(launch_counted(LK_AUX, st, [&] { k_norm2_final<<<B, 32, 0, st>>>(part, nb, norms); return cudaGetLastError(); }));
    std::vector<double> hn(B);
    CK(cudaMemcpyAsync(hn.data(), norms, sizeof(double) * B, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int s = 0; s < B; ++s)
      if (!(std::fabs(hn[s] - 1.0) <= 1e-8)) return fail(SRE_ENOTNORM, "state %d: ||psi||^2 = %.17g", s, hn[s]);
  }
  rc = run_range(dpsi, N, B, 0, 1ull << N, alpha, n_alpha, g_cache.ws, ws_bytes_for(p, B, prec), sums, st, prec);
  if (rc) return rc;
  std::vector<double> hs((size_t)B * (n_alpha + 2));
  CK(cudaMemcpyAsync(hs.data(), sums, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return sre_finalize(hs.data(), N, B, alpha, n_alpha, out_M, out_ln);
}

}  // namespace

// ==========================================================================================
// exported C ABI
// ==========================================================================================
extern "C" {

const char* sre_status_string(int code) {
  switch (code) {
    case SRE_OK: return "ok";
    case SRE_EINVAL: return "invalid argument";
    case SRE_ERANGE: return "size out of range";
    case SRE_ENOTNORM: return "state not normalised";
    case SRE_EWORKSPACE: return "workspace too small";
    case SRE_ENOMEM: return "device allocation failed";
    case SRE_ECUDA: return "CUDA error";
    case SRE_EINTERNAL: return "internal error";
    case SRE_ENODEV: return "no sm_100 device";
  }
  return "unknown status";
}

const char* sre_last_error(void) { return g_err; }

int sre_version(void) { return 100; }

size_t sre_workspace_size(int N, int B, int n_alpha) {
  if (N < 1 || N > SRE_MAX_N || B < 1 || n_alpha < 1 || n_alpha > SRE_MAX_ALPHA) return 0;
  Dev d;  // plan does not depend on the device
  Plan p;
  make_plan(N, d, p);
  return ws_bytes_for(p, B);
}

int sre_exact(const void* psi, int N, const double* alpha, int n_alpha, double* out_M, double* out_lost_norm) {
  g_err[0] = 0;
  return exact_impl(psi, N, 1, alpha, n_alpha, out_M, out_lost_norm);
}

int sre_exact_batched(const void* psi, int N, int B, const double* alpha, int n_alpha, double* out_M,
                      double* out_lost_norm) {
  g_err[0] = 0;
  return exact_impl(psi, N, B, alpha, n_alpha, out_M, out_lost_norm);
}

size_t sre_workspace_size_ex(int N, int B, int n_alpha, int precision) {
  if (N < 1 || N > SRE_MAX_N || B < 1 || n_alpha < 1 || n_alpha > SRE_MAX_ALPHA) return 0;
  if (precision != SRE_FP64 && precision != SRE_FP32) return 0;
  Dev d;
  Plan p;
  make_plan(N, d, p);
  return ws_bytes_for(p, B, precision);
}

int sre_exact_ex(const void* psi, int N, int B, const double* alpha, int n_alpha, int precision, double* out_M,
                 double* out_lost_norm) {
  g_err[0] = 0;
  return exact_impl(psi, N, B, alpha, n_alpha, out_M, out_lost_norm, precision);
}

int sre_partial_sums_ex(const void* psi, int N, int B, uint64_t a_begin, uint64_t a_end, const double* alpha,
                        int n_alpha, int precision, void* workspace, size_t ws_bytes, double* sums_dev, void* stream) {
  g_err[0] = 0;
  if (precision != SRE_FP64 && precision != SRE_FP32) return fail(SRE_EINVAL, "precision %d", precision);
  int rc = validate_common(psi, N, B, alpha, n_alpha);
  if (rc) return rc;
  if (!workspace) return fail(SRE_EINVAL, "workspace is NULL");
  if (!sums_dev) return fail(SRE_EINVAL, "sums_dev is NULL");
  if (a_begin > a_end || a_end > (1ull << N)) return fail(SRE_ERANGE, "range [%llu, %llu) outside [0, 2^%d]",
                                                          (unsigned long long)a_begin, (unsigned long long)a_end, N);
  bool dv = false;
  is_device_ptr(psi, dv);
  if (!dv) return fail(SRE_EINVAL, "psi must be a device pointer");
  return run_range(reinterpret_cast<const double2*>(psi), N, B, a_begin, a_end, alpha, n_alpha,
                   reinterpret_cast<char*>(workspace), ws_bytes, sums_dev, reinterpret_cast<cudaStream_t>(stream),
                   precision);
}

int sre_x_string_sums(const void* psi, int N, const uint64_t* a_list, int n_a, const double* alpha, int n_alpha,
                      void* workspace, size_t ws_bytes, double* out_dev, void* stream) {
  g_err[0] = 0;
  int rc = validate_common(psi, N, 1, alpha, n_alpha);
  if (rc) return rc;
  if (!a_list || !workspace || !out_dev) return fail(SRE_EINVAL, "NULL argument");
  if (n_a < 0) return fail(SRE_EINVAL, "n_a=%d", n_a);
  for (int i = 0; i < n_a; ++i)
    if (a_list[i] >= (1ull << N)) return fail(SRE_ERANGE, "a_list[%d]=%llu >= 2^%d", i, (unsigned long long)a_list[i], N);
  bool dv = false;
  is_device_ptr(psi, dv);
  if (!dv) return fail(SRE_EINVAL, "psi must be a device pointer");
  const char* lm = getenv("SRE_LIST");     // SRE_LIST=0: per-X-string ranges (comparison)
  if (N - 1 <= MID_MAX_T && n_a > 0 && !(lm && lm[0] == '0')) {   // one launch per sweep for the list
    Dev d;
    rc = get_dev(d);
    if (rc) return rc;
    Plan p;
    make_plan(N, d, p, 1);
    const size_t list_off = (size_t)kListMax * NACC * sizeof(double);   // after the item slots
    if (ws_bytes < list_off + (size_t)kListMax * sizeof(uint64_t) || ws_bytes < ws_bytes_for(p, 1))
      return fail(SRE_EWORKSPACE, "workspace %zu too small for list mode", ws_bytes);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint64_t* dl = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(workspace) + list_off);
    for (int c0 = 0; c0 < n_a; c0 += kListMax) {
      const int cn = (n_a - c0) < kListMax ? (n_a - c0) : kListMax;
      CK(cudaMemcpyAsync(dl, a_list + c0, sizeof(uint64_t) * cn, cudaMemcpyHostToDevice, st));
      rc = run_list(reinterpret_cast<const double2*>(psi), N, dl, cn, alpha, n_alpha, reinterpret_cast<char*>(workspace),
                    out_dev + (size_t)c0 * (n_alpha + 2), st);
      if (rc) return rc;
    }
    return SRE_OK;
  }
  for (int i = 0; i < n_a; ++i) {
    rc = run_range(reinterpret_cast<const double2*>(psi), N, 1, a_list[i], a_list[i] + 1, alpha, n_alpha,
                   reinterpret_cast<char*>(workspace), ws_bytes, out_dev + (size_t)i * (n_alpha + 2),
                   reinterpret_cast<cudaStream_t>(stream));
    if (rc) return rc;
  }
  return SRE_OK;
}

int sre_partial_sums(const void* psi, int N, int B, uint64_t a_begin, uint64_t a_end, const double* alpha, int n_alpha,
                     void* workspace, size_t ws_bytes, double* sums_dev, void* stream) {
  g_err[0] = 0;
  int rc = validate_common(psi, N, B, alpha, n_alpha);
  if (rc) return rc;
  if (!workspace) return fail(SRE_EINVAL, "workspace is NULL");
  if (!sums_dev) return fail(SRE_EINVAL, "sums_dev is NULL");
  if (a_begin > a_end || a_end > (1ull << N)) return fail(SRE_ERANGE, "range [%llu, %llu) outside [0, 2^%d]",
                                                          (unsigned long long)a_begin, (unsigned long long)a_end, N);
  bool dv = false;
  is_device_ptr(psi, dv);
  if (!dv) return fail(SRE_EINVAL, "psi must be a device pointer");
  is_device_ptr(sums_dev, dv);
  if (!dv) return fail(SRE_EINVAL, "sums_dev must be a device pointer");
  return run_range(reinterpret_cast<const double2*>(psi), N, B, a_begin, a_end, alpha, n_alpha,
                   reinterpret_cast<char*>(workspace), ws_bytes, sums_dev, reinterpret_cast<cudaStream_t>(stream));
}

int sre_finalize(const double* sums, int N, int B, const double* alpha, int n_alpha, double* out_M,
                 double* out_lost_norm) {
  if (!sums || !alpha || !out_M) return fail(SRE_EINVAL, "NULL argument");
  if (N < 1 || N > SRE_MAX_N || B < 1) return fail(SRE_ERANGE, "N=%d B=%d", N, B);
  if (n_alpha < 1 || n_alpha > SRE_MAX_ALPHA) return fail(SRE_EINVAL, "n_alpha=%d", n_alpha);
  const double D = std::ldexp(1.0, N);
  for (int s = 0; s < B; ++s) {
    const double* r = sums + (size_t)s * (n_alpha + 2);
    for (int i = 0; i < n_alpha; ++i) {
      if (alpha[i] == 1.0)
        out_M[(size_t)s * n_alpha + i] = -(r[n_alpha + 1] / std::log(2.0)) / D;  // reading C4
      else
        out_M[(size_t)s * n_alpha + i] = std::log2(r[i] / D) / (1.0 - alpha[i]);  // Eq. (2)
    }
    if (out_lost_norm) out_lost_norm[s] = 1.0 - r[n_alpha] / D;
  }
  return SRE_OK;
}

int sre_norm2(const void* psi, int N, int B, double* out_dev, void* stream) {
  if (!psi || !out_dev) return fail(SRE_EINVAL, "NULL argument");
  if (N < 1 || N > SRE_MAX_N || B < 1) return fail(SRE_ERANGE, "N=%d B=%d", N, B);
  // single-block-per-state reduction straight into out_dev (no workspace needed)
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  dim3 g(1, B);
  CK(launch_counted(LK_AUX, st, [&] {
    k_norm2_partial<<<g, 1024, 0, st>>>(reinterpret_cast<const double2*>(psi), N, out_dev);
    return cudaGetLastError();
  }));
  return SRE_OK;
}

int sre_chi(const void* psi, int N, uint64_t a, double* chi_dev, void* stream) {
  g_err[0] = 0;
  double one = 2.0;
  int rc = validate_common(psi, N, 1, &one, 1);
  if (rc) return rc;
  if (!chi_dev) return fail(SRE_EINVAL, "chi_dev is NULL");
  if (a >= (1ull << N)) return fail(SRE_ERANGE, "a out of range");
  Dev d;
  rc = get_dev(d);
  if (rc) return rc;
  Plan p;
  make_plan(N, d, p, 1);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double2* dpsi = reinterpret_cast<const double2*>(psi);
  Alphas al;
  memset(&al, 0, sizeof(al));
  al.n = 1;
  cudaError_t e = cudaSuccess;
  if (p.kind == SMALL) {
    e = launch_small<double, false, true>(p.T, dpsi, N, 1, 1, a, 1, al, nullptr, chi_dev, st, nullptr);
  } else if (p.kind == MID) {
    e = launch_mid<double, false, true>(p.T, dpsi, N, 1, 1, a, 1, al, nullptr, chi_dev, st, nullptr);
  } else {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    Cache& g_cache = g_caches[d.id];
    rc = cache_get(&g_cache.ws, &g_cache.ws_bytes, ws_bytes_for(p, 1));
    if (rc) return rc;
    double* slab = reinterpret_cast<double*>(g_cache.ws + off_slab(p, 1));
    if (p.staged && a >= p.amin && a % 8 == 0) {
      // the production kernels of the sums (staged / streamed pass A + TMA pass B, kcount = 1): the pass-B
      // epilogue decodes every output into chi_b(a) (Alphas::chi); its sums land in scratch slots
      double* partial = reinterpret_cast<double*>(g_cache.ws);
      al.chi = chi_dev;
      al.chi_a0 = a;
      e = launch_passA10s<double>(p, d, dpsi, a, 1, slab, st);
      if (e == cudaSuccess) e = launch_passBp<double, false>(p, d, 1, slab, al, partial, st);
    } else {   // generic head (a < 2^L or unaligned): the kernels those X-strings take in the sums
      e = launch_passA<double>(p, dpsi, a, 1, slab, st);
      if (e == cudaSuccess) e = launch_passB<double, false, true>(p, a, 1, slab, al, nullptr, chi_dev, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (e != cudaSuccess) return fail(SRE_ECUDA, "sre_chi: %s", cudaGetErrorString(e));
  return SRE_OK;
}

int sre_pauli_spectrum(const void* psi, int N, uint64_t a_begin, uint64_t a_end, uint64_t* hist_dev, void* workspace,
                       size_t ws_bytes, void* stream) {
  g_err[0] = 0;
  double two = 2.0;
  int rc = validate_common(psi, N, 1, &two, 1);
  if (rc) return rc;
  if (!hist_dev || !workspace) return fail(SRE_EINVAL, "NULL argument");
  if (a_begin > a_end || a_end > (1ull << N)) return fail(SRE_ERANGE, "range [%llu, %llu) outside [0, 2^%d]",
                                                          (unsigned long long)a_begin, (unsigned long long)a_end, N);
  bool dv = false;
  is_device_ptr(psi, dv);
  if (!dv) return fail(SRE_EINVAL, "psi must be a device pointer");
  Dev d;
  rc = get_dev(d);
  if (rc) return rc;
  Plan p;
  make_plan(N, d, p, a_end - a_begin);
  if (ws_bytes < ws_bytes_for(p, 1)) return fail(SRE_EWORKSPACE, "workspace %zu < required %zu", ws_bytes, ws_bytes_for(p, 1));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long* h = reinterpret_cast<unsigned long long*>(hist_dev);
  CK(cudaMemsetAsync(h, 0, sizeof(unsigned long long) * SPEC_BINS, st));
  const uint64_t count = a_end - a_begin;
  if (count == 0) return SRE_OK;
  if (p.kind == TWOPASS) {   // pass-B epilogues bin the final values; sums go to a scratch tail
    const size_t need = ws_bytes_for(p, 1) + 256;
    if (ws_bytes < need) return fail(SRE_EWORKSPACE, "workspace %zu < required %zu", ws_bytes, need);
    double* scratch = reinterpret_cast<double*>(reinterpret_cast<char*>(workspace) + ws_bytes_for(p, 1));
    return run_range(reinterpret_cast<const double2*>(psi), N, 1, a_begin, a_end, &two, 1,
                     reinterpret_cast<char*>(workspace), ws_bytes_for(p, 1), scratch, st, SRE_FP64, h);
  }
  const std::vector<Sweep> sw = make_sweeps(&two, 1);
  const double2* dpsi = reinterpret_cast<const double2*>(psi);
  double* partial = reinterpret_cast<double*>(workspace);   // the alpha sums are computed and ignored
  cudaError_t e;
  if (p.kind == SMALL) {
    const int G = p.T >= 5 ? 32 : (1 << p.T);
    const int gx = std::min<int>(pick_gx(count, 256 / G, 1, occupancy_small(p.T, d)), (int)p.slots);
    e = launch_small<double, true, false>(p.T, dpsi, N, 1, gx, a_begin, count, sw[0].al, partial, nullptr, st, nullptr, h);
  } else {
    const int gx = std::min<int>(pick_gx(count, 256 >> (p.T - 5), 1, d.sms), (int)p.slots);
    e = launch_mid<double, true, false>(p.T, dpsi, N, 1, gx, a_begin, count, sw[0].al, partial, nullptr, st, nullptr, h);
  }
  if (e != cudaSuccess) return fail(SRE_ECUDA, "spectrum: %s", cudaGetErrorString(e));
  return SRE_OK;
}

uint64_t sre_launch_count(void) { return g_launches.load(); }

int sre_profile_begin(int stride) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  if (stride < 1) return fail(SRE_EINVAL, "stride %d < 1", stride);
  for (int k = 0; k < LK_N; ++k) {
    for (auto& pr : g_prof.timed[k]) { g_prof.pool.push_back(pr.first); g_prof.pool.push_back(pr.second); }
    g_prof.timed[k].clear();
    g_prof.launched[k] = 0;
  }
  g_prof.stride = stride;
  g_prof.on = true;
  return SRE_OK;
}

int sre_profile_end(double* ms_sum, uint64_t* n_timed, uint64_t* n_launched) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = false;
  for (int k = 0; k < LK_N; ++k) {
    double acc = 0.0;
    for (auto& pr : g_prof.timed[k]) {
      float ms = 0.f;
      CK(cudaEventSynchronize(pr.second));
      CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
      acc += ms;
    }
    if (ms_sum) ms_sum[k] = acc;
    if (n_timed) n_timed[k] = g_prof.timed[k].size();
    if (n_launched) n_launched[k] = g_prof.launched[k];
  }
  return SRE_OK;
}

}  // extern "C"
