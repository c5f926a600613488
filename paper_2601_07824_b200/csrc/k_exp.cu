// k_exp.cu -- FP64-only experimental paths: the fused persistent kernel (SRE_FUSED=1) and the
// TMEM pass-B path (SRE_TMEM=1).  Both are correct (tests/test_gpu_parity.py under the env vars)
// and measured slower than the default staged path.
#define SRE_FAMILY_EXP
#include "launch.cuh"

namespace sre_host {

template <int N>
cudaError_t launch_passA_tmem_t(const Dev& d, const double2* psi, uint64_t a_first, int kcount, double* ws,
                                cudaStream_t st) {
  constexpr int L = N == 20 ? 11 : 10;
  constexpr int SMEM = N == 20 ? PA11_SMEM : PA10_SMEM;
  auto kern = [] { if constexpr (N == 20) return k_passA11t<20>; else return k_passA10s<N, true>; }();
  static bool init = false;
  if (!init) {
    cudaError_t e = set_smem(kern, SMEM);
    if (e != cudaSuccess) return e;
    init = true;
  }
  const int groups = (kcount + 7) / 8;
  const uint64_t items = (uint64_t)groups << (N - 1 - L);
  const unsigned grid = (unsigned)(items < (uint64_t)d.sms ? items : (uint64_t)d.sms);
  return launch_counted(LK_PASSA, st, [&] {
    kern<<<grid, 256, SMEM, st>>>(psi, a_first, kcount, groups, ws);
    return cudaGetLastError();
  });
}

template <int N, bool A2>
cudaError_t launch_passB_tmem_t(const Dev& d, int kcount, const double* ws, const Alphas& al, double* partial,
                                cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaError_t e = set_smem(k_passBt8<N, A2>, PB8_SMEM);
    if (e != cudaSuccess) return e;
    init = true;
  }
  return launch_counted(LK_PASSB, st, [&] {
    k_passBt8<N, A2><<<d.sms, 128, PB8_SMEM, st>>>(kcount, ws, al, partial);
    return cudaGetLastError();
  });
}

cudaError_t launch_tmem_pair(const Plan& p, const Dev& d, bool a2, const double2* psi, uint64_t a_first, int kcount,
                             double* ws, const Alphas& al, double* partial, cudaStream_t st) {
  cudaError_t e;
  if (p.N == 20) {
    e = launch_passA_tmem_t<20>(d, psi, a_first, kcount, ws, st);
    if (e == cudaSuccess) e = a2 ? launch_passB_tmem_t<20, true>(d, kcount, ws, al, partial, st)
                                 : launch_passB_tmem_t<20, false>(d, kcount, ws, al, partial, st);
  } else {
    e = launch_passA_tmem_t<19>(d, psi, a_first, kcount, ws, st);
    if (e == cudaSuccess) e = a2 ? launch_passB_tmem_t<19, true>(d, kcount, ws, al, partial, st)
                                 : launch_passB_tmem_t<19, false>(d, kcount, ws, al, partial, st);
  }
  return e;
}

template <int N, bool A2>
cudaError_t launch_fused_t(const Dev& d, const double2* psi, uint64_t a_first, uint64_t count, double* ws,
                           FusedCtl* ctl, const Alphas& al, double* partial, cudaStream_t st) {
  static bool init = false;
  if (!init) {
    cudaError_t e = set_smem(k_fused<N, A2>, FZ_SMEM);
    if (e != cudaSuccess) return e;
    init = true;
  }
  cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(FusedCtl), st);
  if (e != cudaSuccess) return e;
  return launch_counted(LK_FUSED, st, [&] {
    void* args[] = {(void*)&psi, (void*)&a_first, (void*)&count, (void*)&ws, (void*)&ctl, (void*)&al, (void*)&partial};
    return cudaLaunchCooperativeKernel((const void*)k_fused<N, A2>, dim3(d.sms), dim3(256), args, FZ_SMEM, st);
  });
}

template <bool A2>
cudaError_t launch_fused(const Plan& p, const Dev& d, const double2* psi, uint64_t a_first, uint64_t count,
                         double* ws, FusedCtl* ctl, const Alphas& al, double* partial, cudaStream_t st) {
  switch (p.N) {
#define C_(n) case n: return launch_fused_t<n, A2>(d, psi, a_first, count, ws, ctl, al, partial, st);
    C_(15) C_(16) C_(17) C_(18) C_(19) C_(20)
#undef C_
  }
  return cudaErrorInvalidValue;
}

template SRE_SIG_FUSED(true);
template SRE_SIG_FUSED(false);

}  // namespace sre_host
