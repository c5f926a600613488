// launch.cuh -- host-side launch templates shared by the kernel-family translation units.
// Each family .cu file (k_small.cu, k_mid.cu, k_generic.cu, k_stageA.cu, k_stageB.cu)
// explicitly instantiates its dispatchers; sre_api.cu sees them as extern templates, so the
// kernels compile once each and in parallel (paper_2601_07824_b200/_build.py).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/sre.h"
#include "sre_kernels.cuh"

namespace sre_host {
using namespace sre;

enum LaunchKind { LK_SINGLE = 0, LK_PASSA = 1, LK_PASSB = 2, LK_AUX = 3, LK_FUSED = 4, LK_N = 5 };

struct Prof {
  std::mutex mu;
  bool on = false;
  int stride = 1;
  uint64_t launched[LK_N] = {0, 0, 0, 0, 0};
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed[LK_N];
};
extern Prof g_prof;
extern std::atomic<uint64_t> g_launches;
cudaEvent_t prof_event();

// Wraps one kernel launch: counts it, and when profiling, brackets every stride-th launch of
// its kind with CUDA events on the launching stream.
template <class F>
cudaError_t launch_counted(int kind, cudaStream_t st, F&& f) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof.on) return f();
  std::lock_guard<std::mutex> lk(g_prof.mu);
  const bool sample = (g_prof.launched[kind]++ % (uint64_t)g_prof.stride) == 0;
  if (!sample) return f();
  cudaEvent_t a = prof_event(), b = prof_event();
  cudaEventRecord(a, st);
  cudaError_t e = f();
  cudaEventRecord(b, st);
  g_prof.timed[kind].push_back({a, b});
  return e;
}

struct Dev {
  int id = -1, sms = 0, major = 0, minor = 0;
};

enum Kind { SMALL = 0, MID = 1, TWOPASS = 2 };

struct Plan {
  int N = 0, T = 0, kind = 0;
  int L = 0, H = 0, CB = 0, TP = 0, K = 0;  // two-pass
  int unitsA = 0, unitsB = 0, blkB = 0;
  size_t slab_doubles = 0;  // K * 2^N
  size_t slots = 0;         // partial slots per state
  bool staged = false;      // staged (N = 15..20) or streamed (N = 21..25) pass A + TMA-fed pass B
  uint64_t amin = 0;        // first X-string the staged / streamed kernels accept (a_h != 0)
  int KG = 0;               // 8-X-string groups per staged / streamed launch pair
};

// ------------------------------------------------------------------------------------------
// launchers (template dispatch)
// ------------------------------------------------------------------------------------------
template <class V, int T, bool A2, bool DBG>
cudaError_t launch_small_t(const typename Cx<V>::T* psi, int N, int B, int gx, uint64_t a0, uint64_t count, const Alphas& al,
                           double* partial, double* chi, cudaStream_t st, const uint64_t* alist,
                           unsigned long long* hist = nullptr) {
  dim3 grid(gx, B);
  return launch_counted(LK_SINGLE, st, [&] {
    k_small<T, A2, DBG, V><<<grid, 256, 0, st>>>(psi, N, a0, count, al, partial, chi, alist, hist);
    return cudaGetLastError();
  });
}

template <class V, bool A2, bool DBG>
cudaError_t launch_small(int T, const typename Cx<V>::T* psi, int N, int B, int gx, uint64_t a0, uint64_t count, const Alphas& al,
                         double* partial, double* chi, cudaStream_t st, const uint64_t* alist,
                           unsigned long long* hist = nullptr) {
  switch (T) {
#define C_(t) case t: return launch_small_t<V, t, A2, DBG>(psi, N, B, gx, a0, count, al, partial, chi, st, alist, hist);
    C_(0) C_(1) C_(2) C_(3) C_(4) C_(5) C_(6) C_(7) C_(8) C_(9) C_(10)
#undef C_
  }
  return cudaErrorInvalidValue;
}

constexpr int SMEM_128K = 2 * padded(32 * 256) * 8;  // 2 planes x (2^T + pad) x UPC units

template <class K>
cudaError_t set_smem(K kern, int bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
// Raise a kernel's dynamic shared-memory limit once per device (bit d of `mask`): the attribute is per
// device context, so a process that switches devices must set it again there.
template <class K>
cudaError_t set_smem_once(K kern, int bytes, uint64_t& mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && ((mask >> dev) & 1ull)) return cudaSuccess;
  e = set_smem(kern, bytes);
  if (e == cudaSuccess && dev < 64) mask |= 1ull << dev;
  return e;
}

template <class V, int T, bool A2, bool DBG>
cudaError_t launch_mid_t(const typename Cx<V>::T* psi, int N, int B, int gx, uint64_t a0, uint64_t count, const Alphas& al,
                         double* partial, double* chi, cudaStream_t st, const uint64_t* alist,
                           unsigned long long* hist = nullptr) {
  static uint64_t init_mask = 0;   // per device: the attribute belongs to the device context
  if constexpr (T == 13 && !DBG) {  // N = 14 sweeps: ring-fed generation (k_midr) unless SRE_MIDR=0
    static const bool ring = [] { const char* e = getenv("SRE_MIDR"); return !(e && e[0] == '0'); }();
    if (ring && !alist) {
      constexpr int smem = 2 * padded(1 << T) * (int)sizeof(double) + MR_NS * 1024 * (int)sizeof(typename Cx<V>::T);
      static uint64_t init_mask_r = 0;
      cudaError_t e = set_smem_once(k_midr<T, A2, V>, smem, init_mask_r);
      if (e != cudaSuccess) return e;
      dim3 grid(gx, B);
      return launch_counted(LK_SINGLE, st, [&] {
        k_midr<T, A2, V><<<grid, 256, smem, st>>>(psi, N, a0, count, al, partial, hist);
        return cudaGetLastError();
      });
    }
  }
  {
    cudaError_t e = set_smem_once(k_mid<T, A2, DBG, V>, SMEM_128K, init_mask);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(gx, B);
  return launch_counted(LK_SINGLE, st, [&] {
    k_mid<T, A2, DBG, V><<<grid, 256, SMEM_128K, st>>>(psi, N, a0, count, al, partial, chi, alist, hist);
    return cudaGetLastError();
  });
}

template <class V, bool A2, bool DBG>
cudaError_t launch_mid(int T, const typename Cx<V>::T* psi, int N, int B, int gx, uint64_t a0, uint64_t count, const Alphas& al,
                       double* partial, double* chi, cudaStream_t st, const uint64_t* alist,
                           unsigned long long* hist = nullptr) {
  switch (T) {
    case 11: return launch_mid_t<V, 11, A2, DBG>(psi, N, B, gx, a0, count, al, partial, chi, st, alist, hist);
    case 12: return launch_mid_t<V, 12, A2, DBG>(psi, N, B, gx, a0, count, al, partial, chi, st, alist, hist);
    case 13: return launch_mid_t<V, 13, A2, DBG>(psi, N, B, gx, a0, count, al, partial, chi, st, alist, hist);
  }
  return cudaErrorInvalidValue;
}

template <class V, int L>
cudaError_t launch_passA_t(const typename Cx<V>::T* psi, int N, uint64_t a0, int kcount, V* ws, int units, cudaStream_t st) {
  static uint64_t init_mask = 0;   // per device: the attribute belongs to the device context
  {
    cudaError_t e = set_smem_once(k_passA<L, V>, SMEM_128K, init_mask);
    if (e != cudaSuccess) return e;
  }
  const uint64_t items = (uint64_t)kcount << (N - 1 - L);
  const unsigned grid = (unsigned)((items + units - 1) / units);
  return launch_counted(LK_PASSA, st, [&] {
    k_passA<L, V><<<grid, 256, SMEM_128K, st>>>(psi, N, a0, kcount, ws);
    return cudaGetLastError();
  });
}

template <class V>
cudaError_t launch_passA(const Plan& p, const typename Cx<V>::T* psi, uint64_t a0, int kcount, V* ws, cudaStream_t st) {
  switch (p.L) {
    case 10: return launch_passA_t<V, 10>(psi, p.N, a0, kcount, ws, p.unitsA, st);
    case 11: return launch_passA_t<V, 11>(psi, p.N, a0, kcount, ws, p.unitsA, st);
    case 12: return launch_passA_t<V, 12>(psi, p.N, a0, kcount, ws, p.unitsA, st);
    case 13: return launch_passA_t<V, 13>(psi, p.N, a0, kcount, ws, p.unitsA, st);
  }
  return cudaErrorInvalidValue;
}

template <class V, int TP, int CB, bool A2, bool DBG>
cudaError_t launch_passB_t(const Plan& p, uint64_t a0, int kcount, const V* ws, const Alphas& al, double* partial,
                           double* chi, cudaStream_t st) {
  constexpr int BLK = TP >= 14 ? 512 : 256;
  constexpr int SM = padded(BLK * 32) * 8;
  static uint64_t init_mask = 0;   // per device: the attribute belongs to the device context
  {
    cudaError_t e = set_smem_once(k_passB<TP, CB, A2, DBG, V>, SM, init_mask);
    if (e != cudaSuccess) return e;
  }
  const uint64_t items = (uint64_t)kcount * 2 * (1ull << (p.L - CB));
  const unsigned grid = (unsigned)((items + p.unitsB - 1) / p.unitsB);
  return launch_counted(LK_PASSB, st, [&] {
    k_passB<TP, CB, A2, DBG, V><<<grid, BLK, SM, st>>>(p.N, p.L, a0, kcount, ws, al, partial, chi);
    return cudaGetLastError();
  });
}

template <class V, bool A2, bool DBG>
cudaError_t launch_passB(const Plan& p, uint64_t a0, int kcount, const V* ws, const Alphas& al, double* partial,
                         double* chi, cudaStream_t st) {
  const int key = p.TP * 16 + p.CB;
  switch (key) {
#define C_(tp, cb) case tp * 16 + cb: return launch_passB_t<V, tp, cb, A2, DBG>(p, a0, kcount, ws, al, partial, chi, st);
    C_(10, 6) C_(11, 6) C_(12, 6) C_(13, 6) C_(13, 5) C_(13, 4) C_(13, 3) C_(13, 2) C_(14, 2)
#undef C_
  }
  return cudaErrorInvalidValue;
}

template <class V, int N, bool ROWM = false>
cudaError_t launch_passA10s_t(const Dev& d, const typename Cx<V>::T* psi, uint64_t a_first, int kcount, V* ws,
                              cudaStream_t st) {
  static uint64_t init_mask = 0;   // per device: the attribute belongs to the device context
  {
    cudaError_t e = set_smem_once(k_passA10s<N, V, ROWM>, PA10_SMEM, init_mask);
    if (e != cudaSuccess) return e;
  }
  const int groups = (kcount + 7) / 8;
  const uint64_t items = (uint64_t)groups << (N - 11);
  const unsigned grid = (unsigned)(items < (uint64_t)d.sms ? items : (uint64_t)d.sms);
  return launch_counted(LK_PASSA, st, [&] {
    k_passA10s<N, V, ROWM><<<grid, 256, PA10_SMEM, st>>>(psi, a_first, kcount, groups, ws);
    return cudaGetLastError();
  });
}

template <class V, int N, int L>
cudaError_t launch_passAs_t(const Dev& d, const typename Cx<V>::T* psi, uint64_t a_first, int kcount, V* ws,
                            cudaStream_t st) {
  static uint64_t init_mask = 0;   // per device: the attribute belongs to the device context
  {
    cudaError_t e = set_smem_once(k_passAs<N, L, V>, pas_smem(L), init_mask);
    if (e != cudaSuccess) return e;
  }
  const uint64_t units = (uint64_t)kcount << (N - 1 - L);
  const uint64_t ctas = (units + (256 >> (L - 5)) - 1) / (256 >> (L - 5));
  const unsigned grid = (unsigned)(ctas < (uint64_t)d.sms ? ctas : (uint64_t)d.sms);
  return launch_counted(LK_PASSA, st, [&] {
    k_passAs<N, L, V><<<grid, 256, pas_smem(L), st>>>(psi, a_first, kcount, ws);
    return cudaGetLastError();
  });
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

template <int N>
cudaError_t launch_passAw_t(const Dev& d, const double2* psi, uint64_t a_first, int kcount, double* ws, cudaStream_t st) {
  static const bool ts = [] { const char* e = getenv("SRE_PAW_TMA"); return !(e && e[0] == '0'); }();
  static uint64_t init_mask = 0, init_mask_ts = 0;
  {
    cudaError_t e = ts ? set_smem_once(k_passAw<N, true>, PAW_SMEM, init_mask_ts) : set_smem_once(k_passAw<N, false>, PAW_SMEM, init_mask);
    if (e != cudaSuccess) return e;
  }
  // TMA store map: row-plane r = (2k + p) 2^H + y_h as the 64 x 64 matrix [t][j], boxes {16, 64, 1}
  CUtensorMap tm;
  std::memset(&tm, 0, sizeof(tm));
  if (ts) {
    auto enc = tensor_map_encoder();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {64, 64, (cuuint64_t)kcount << (N - 12)};
    const cuuint64_t strides[2] = {64 * sizeof(double), 4096 * sizeof(double)};
    const cuuint32_t box[3] = {16, 64, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ws, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const uint64_t groups = (uint64_t)(kcount + 3) / 4;
  const uint64_t items = groups << (N - 13);                         // (row, group of 4 X-strings)
  const unsigned grid = (unsigned)(items < (uint64_t)d.sms ? items : (uint64_t)d.sms);
  const uint64_t gmagic = ((1ull << 40) + groups - 1) / groups;
  return launch_counted(LK_PASSA, st, [&] {
    if (ts) k_passAw<N, true><<<grid, 256, PAW_SMEM, st>>>(psi, a_first, kcount, gmagic, ws, tm);
    else k_passAw<N, false><<<grid, 256, PAW_SMEM, st>>>(psi, a_first, kcount, gmagic, ws, tm);
    return cudaGetLastError();
  });
}

template <class V>
cudaError_t launch_passA10s(const Plan& p, const Dev& d, const typename Cx<V>::T* psi, uint64_t a_first, int kcount,
                            V* ws, cudaStream_t st) {
  constexpr bool F64 = std::is_same<V, double>::value;   // FP64 N >= 17: row-major workspace planes
  if constexpr (F64) {   // FP64 N = 21..24: radix-64 pass A (TMEM-parked plane B), row-major rows
    if (p.N >= 21 && p.N <= 24) {
      switch (p.N) {
        case 21: return launch_passAw_t<21>(d, psi, a_first, kcount, ws, st);
        case 22: return launch_passAw_t<22>(d, psi, a_first, kcount, ws, st);
        case 23: return launch_passAw_t<23>(d, psi, a_first, kcount, ws, st);
        case 24: return launch_passAw_t<24>(d, psi, a_first, kcount, ws, st);
      }
    }
  }
  switch (p.N) {
    case 21: return launch_passAs_t<V, 21, 12>(d, psi, a_first, kcount, ws, st);
    case 22: return launch_passAs_t<V, 22, 12>(d, psi, a_first, kcount, ws, st);
    case 23: return launch_passAs_t<V, 23, 12>(d, psi, a_first, kcount, ws, st);
    case 24: return launch_passAs_t<V, 24, 12>(d, psi, a_first, kcount, ws, st);
    case 25: return launch_passAs_t<V, 25, 13>(d, psi, a_first, kcount, ws, st);
    case 15: return launch_passA10s_t<V, 15>(d, psi, a_first, kcount, ws, st);   // slab-major tiles for k_passBt
    case 16: return launch_passA10s_t<V, 16>(d, psi, a_first, kcount, ws, st);
    case 17: return launch_passA10s_t<V, 17, F64>(d, psi, a_first, kcount, ws, st);
    case 18: return launch_passA10s_t<V, 18, F64>(d, psi, a_first, kcount, ws, st);
    case 19: return launch_passA10s_t<V, 19, F64>(d, psi, a_first, kcount, ws, st);
    case 20: return launch_passA10s_t<V, 20, F64>(d, psi, a_first, kcount, ws, st);
  }
  return cudaErrorInvalidValue;
}

template <class V, int TP, int CB, bool A2>
cudaError_t launch_passBt_t(const Plan& p, const Dev& d, int kcount, const V* ws, const Alphas& al,
                            double* partial, cudaStream_t st) {
  static uint64_t init_mask = 0;   // per device: the attribute belongs to the device context
  {
    cudaError_t e = set_smem_once(k_passBt<TP, CB, A2, V>, pbt_smem(TP), init_mask);
    if (e != cudaSuccess) return e;
  }
  const unsigned grid = (unsigned)d.sms;
  return launch_counted(LK_PASSB, st, [&] {
    k_passBt<TP, CB, A2, V><<<grid, 256, pbt_smem(TP), st>>>(p.N, kcount, ws, al, partial);
    return cudaGetLastError();
  });
}

template <int CB, int L, bool A2>
cudaError_t launch_passBw_t(const Plan& p, const Dev& d, int kcount, const double* ws, const Alphas& al, double* partial,
                            cudaStream_t st) {
  static uint64_t init_mask = 0;
  {
    cudaError_t e = set_smem_once(k_passBw<CB, L, A2>, PBR_SMEM, init_mask);
    if (e != cudaSuccess) return e;
  }
  constexpr int H = 13 - CB, R = H >= 8 ? 256 : (1 << H);
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {1ull << L, 1ull << H, (cuuint64_t)2 * (cuuint64_t)kcount};
  const cuuint64_t strides[2] = {(1ull << L) * sizeof(double), (1ull << (p.N - 1)) * sizeof(double)};
  const cuuint32_t box[3] = {1u << CB, (cuuint32_t)R, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ws), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  return launch_counted(LK_PASSB, st, [&] {
    k_passBw<CB, L, A2><<<d.sms, 256, PBR_SMEM, st>>>(kcount, tm, al, partial);
    return cudaGetLastError();
  });
}

template <class V, bool A2>
cudaError_t launch_passBp(const Plan& p, const Dev& d, int kcount, const V* ws, const Alphas& al, double* partial,
                          cudaStream_t st) {
  if constexpr (std::is_same<V, double>::value) {   // FP64 N = 21..24: radix-64 pass B (one transpose)
    if (p.N >= 21 && p.N <= 24) {
      switch (13 - p.H) {
        case 5: return launch_passBw_t<5, 12, A2>(p, d, kcount, ws, al, partial, st);
        case 4: return launch_passBw_t<4, 12, A2>(p, d, kcount, ws, al, partial, st);
        case 3: return launch_passBw_t<3, 12, A2>(p, d, kcount, ws, al, partial, st);
        case 2: return launch_passBw_t<2, 12, A2>(p, d, kcount, ws, al, partial, st);
      }
    }
    if (p.N >= 17 && p.N <= 20) {
      switch (13 - p.H) {   // FP64 N = 17..20: k_passA10s<ROWM> wrote row-major planes
        case 7: return launch_passBw_t<7, 10, A2>(p, d, kcount, ws, al, partial, st);
        case 6: return launch_passBw_t<6, 10, A2>(p, d, kcount, ws, al, partial, st);
        case 5: return launch_passBw_t<5, 10, A2>(p, d, kcount, ws, al, partial, st);
        case 4: return launch_passBw_t<4, 10, A2>(p, d, kcount, ws, al, partial, st);
      }
    }
  }
  if (p.N >= 21) {     // streamed path: tiles of 2^13 doubles, CB = 13 - H
    switch (13 - p.H) {
      case 7: return launch_passBt_t<V, 13, 7, A2>(p, d, kcount, ws, al, partial, st);
      case 6: return launch_passBt_t<V, 13, 6, A2>(p, d, kcount, ws, al, partial, st);
      case 5: return launch_passBt_t<V, 13, 5, A2>(p, d, kcount, ws, al, partial, st);
      case 4: return launch_passBt_t<V, 13, 4, A2>(p, d, kcount, ws, al, partial, st);
      case 3: return launch_passBt_t<V, 13, 3, A2>(p, d, kcount, ws, al, partial, st);
      case 2: return launch_passBt_t<V, 13, 2, A2>(p, d, kcount, ws, al, partial, st);
    }
    return cudaErrorInvalidValue;
  }
  switch (12 - p.H) {  // slab-major tiles of 2^12 doubles: CB = 12 - H
    case 8: return launch_passBt_t<V, 12, 8, A2>(p, d, kcount, ws, al, partial, st);
    case 7: return launch_passBt_t<V, 12, 7, A2>(p, d, kcount, ws, al, partial, st);
    case 6: return launch_passBt_t<V, 12, 6, A2>(p, d, kcount, ws, al, partial, st);
    case 5: return launch_passBt_t<V, 12, 5, A2>(p, d, kcount, ws, al, partial, st);
    case 4: return launch_passBt_t<V, 12, 4, A2>(p, d, kcount, ws, al, partial, st);
    case 3: return launch_passBt_t<V, 12, 3, A2>(p, d, kcount, ws, al, partial, st);
  }
  return cudaErrorInvalidValue;
}


// ------------------------------------------------------------------------------------------
// explicit instantiations: defined in the family translation units
// ------------------------------------------------------------------------------------------
#define SRE_SIG_SMALL(V, A2, DBG) cudaError_t launch_small<V, A2, DBG>(int, const typename Cx<V>::T*, int, int, int, \
    uint64_t, uint64_t, const Alphas&, double*, double*, cudaStream_t, const uint64_t*, unsigned long long*)
#define SRE_SIG_MID(V, A2, DBG) cudaError_t launch_mid<V, A2, DBG>(int, const typename Cx<V>::T*, int, int, int, \
    uint64_t, uint64_t, const Alphas&, double*, double*, cudaStream_t, const uint64_t*, unsigned long long*)
#define SRE_SIG_PASSA(V) cudaError_t launch_passA<V>(const Plan&, const typename Cx<V>::T*, uint64_t, int, V*, cudaStream_t)
#define SRE_SIG_PASSB(V, A2, DBG) cudaError_t launch_passB<V, A2, DBG>(const Plan&, uint64_t, int, const V*, \
    const Alphas&, double*, double*, cudaStream_t)
#define SRE_SIG_STAGEA(V) cudaError_t launch_passA10s<V>(const Plan&, const Dev&, const typename Cx<V>::T*, uint64_t, \
    int, V*, cudaStream_t)
#define SRE_SIG_STAGEB(V, A2) cudaError_t launch_passBp<V, A2>(const Plan&, const Dev&, int, const V*, const Alphas&, \
    double*, cudaStream_t)
#define SRE_FOR_V_A2_DBG(M, P) P M(double, true, false); P M(double, false, false); P M(float, true, false); \
    P M(float, false, false); P M(double, false, true)
#define SRE_FOR_V(M, P) P M(double); P M(float)
#define SRE_FOR_V_A2(M, P) P M(double, true); P M(double, false); P M(float, true); P M(float, false)

#ifndef SRE_FAMILY_SMALL
SRE_FOR_V_A2_DBG(SRE_SIG_SMALL, extern template);
#endif
#ifndef SRE_FAMILY_MID
SRE_FOR_V_A2_DBG(SRE_SIG_MID, extern template);
#endif
#ifndef SRE_FAMILY_GENERIC
SRE_FOR_V(SRE_SIG_PASSA, extern template);
SRE_FOR_V_A2_DBG(SRE_SIG_PASSB, extern template);
#endif
#ifndef SRE_FAMILY_STAGEA
SRE_FOR_V(SRE_SIG_STAGEA, extern template);
#endif
#ifndef SRE_FAMILY_STAGEB
SRE_FOR_V_A2(SRE_SIG_STAGEB, extern template);
#endif

}  // namespace sre_host
