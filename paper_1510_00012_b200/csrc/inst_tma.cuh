// inst_tma.cuh — host launchers of the variant-2 iteration kernel k_badmm_tma<T, MP, NCH, MODE, DP>
// (ad2_tma.cuh) and of the objective kernel k_cost_member.  Each inst_<dtype>_mp<MP>.cu is one
// AD2_INST_TMA(T, MP) line, so nvcc compiles the (dtype, MP) template sets in parallel.
#pragma once
#include "ad2_launch.cuh"
#include "ad2_tma.cuh"

namespace ad2k {

template <typename T, int MP, int NCH, int DP, int TCC = 0>
struct TmaLaunch {
  using Lay = TmaLayout<T, MP, NCH, DP>;
  template <int MODE>
  static void attr() {
    cudaFuncSetAttribute(k_badmm_tma<T, MP, NCH, MODE, DP, TCC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Lay::CTA_BYTES);
  }
  template <int MODE>
  static void go(const IterArgs<T>& a, int64_t n_items, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)n_items);
    cfg.blockDim = dim3(NWARP * 32);
    cfg.dynamicSmemBytes = Lay::CTA_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = a.pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_badmm_tma<T, MP, NCH, MODE, DP, TCC>, a);
  }
  static void run(int mode, const IterArgs<T>& a, int64_t n_items, cudaStream_t s) {
    static PerDevice once;                 // the smem attribute is per device
    if (once.first()) {
      attr<P1ONLY>(); attr<FUSED>(); attr<P2ONLY>(); attr<P1INIT>(); attr<P2X>(); attr<FUSEDX>();
      attr<GIN>(); attr<GMID>(); attr<GXOUT>();
      once.done();
    }
    switch (mode) {
      case P1ONLY: go<P1ONLY>(a, n_items, s); break;
      case FUSED: go<FUSED>(a, n_items, s); break;
      case P1INIT: go<P1INIT>(a, n_items, s); break;
      case P2X: go<P2X>(a, n_items, s); break;
      case FUSEDX: go<FUSEDX>(a, n_items, s); break;
      case GIN: go<GIN>(a, n_items, s); break;
      case GMID: go<GMID>(a, n_items, s); break;
      case GXOUT: go<GXOUT>(a, n_items, s); break;
      default: go<P2ONLY>(a, n_items, s); break;
    }
  }
};

// shared memory of one CTA (dynamic ring + static tiles): the init-time fit check
template <typename T, int MP>
size_t tma_bytes_impl(int nch, int dp) {
  constexpr int NCH2 = MP < 32 ? 2 : 1;      // two column chunks exist only below 32 rows
  if (nch == 2 && MP < 32) {
    if (dp <= 4) return TmaLayout<T, MP, NCH2, 4>::CTA_BYTES + TmaLayout<T, MP, NCH2, 4>::STATIC_BYTES;
    return TmaLayout<T, MP, NCH2, 16>::CTA_BYTES + TmaLayout<T, MP, NCH2, 16>::STATIC_BYTES;
  }
  if (dp <= 4) return TmaLayout<T, MP, 1, 4>::CTA_BYTES + TmaLayout<T, MP, 1, 4>::STATIC_BYTES;
  return TmaLayout<T, MP, 1, 16>::CTA_BYTES + TmaLayout<T, MP, 1, 16>::STATIC_BYTES;
}

template <typename T, int MP>
void launch_tma_impl(int variant, int mode, int nch, int dp, const IterArgs<T>& a, int64_t n_items, cudaStream_t s) {
  if (variant != 2) return;
  if constexpr (MP < 32) {
    if (nch == 2) {
      if (dp <= 4) TmaLaunch<T, MP, 2, 4>::run(mode, a, n_items, s);
      else TmaLaunch<T, MP, 2, 16>::run(mode, a, n_items, s);
      return;
    }
  }
  if (dp <= 4) {
    TmaLaunch<T, MP, 1, 4>::run(mode, a, n_items, s);
    return;
  }
  if constexpr (sizeof(T) == 4 && MP == 32) {
    if (a.tc) {                                // tensor-core cost (single-member 32-row passes)
      TmaLaunch<T, MP, 1, 16, 1>::run(mode, a, n_items, s);
      return;
    }
  }
  TmaLaunch<T, MP, 1, 16>::run(mode, a, n_items, s);
}

template <typename T>
void launch_cost_member_impl(int dp, const int64_t* off, int64_t N, const int32_t* mem_cl, const T* Y, const T* x,
                             const T* P, double* pm, int m, int d, int ld, cudaStream_t s) {
  if (N == 0) return;
  constexpr int NW = cost_member_warps<T>();
  static PerDeviceInt grid_cap;                        // resident CTAs (grid-stride kernel), per device
  int cap = grid_cap.get();
  if (!cap) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cost_member<T, 16>, 32 * NW, 0);
    cap = nsm * (per > 0 ? per : 1);
    grid_cap.set(cap);
  }
  const int64_t need = (N + NW - 1) / NW;
  const unsigned g = (unsigned)(need < cap ? need : cap);
  if (dp <= 4) k_cost_member<T, 4><<<g, 32 * NW, 0, s>>>(off, N, mem_cl, Y, x, P, pm, m, d, ld);
  else k_cost_member<T, 16><<<g, 32 * NW, 0, s>>>(off, N, mem_cl, Y, x, P, pm, m, d, ld);
}

}  // namespace ad2k

// the entry points ad2.cu declares, specialised for one (T, MP)
template <typename T, int MP>
size_t tma_cta_bytes(int nch, int dp);
template <typename T, int MP>
void launch_warp(int variant, int mode, int nch, int dp, const ad2k::IterArgs<T>& a, int64_t n_items, cudaStream_t s);
template <typename T>
void launch_cost_member(int dp, const int64_t* off, int64_t N, const int32_t* mem_cl, const T* Y, const T* x,
                        const T* P, double* pm, int m, int d, int ld, cudaStream_t s);

#define AD2_INST_TMA(T, MP)                                                                                    \
  template <>                                                                                                  \
  size_t tma_cta_bytes<T, MP>(int nch, int dp) {                                                               \
    return ad2k::tma_bytes_impl<T, MP>(nch, dp);                                                               \
  }                                                                                                            \
  template <>                                                                                                  \
  void launch_warp<T, MP>(int variant, int mode, int nch, int dp, const ad2k::IterArgs<T>& a, int64_t n_items, \
                          cudaStream_t s) {                                                                    \
    ad2k::launch_tma_impl<T, MP>(variant, mode, nch, dp, a, n_items, s);                                       \
  }

#define AD2_INST_COST_MEMBER(T)                                                                                \
  template <>                                                                                                  \
  void launch_cost_member<T>(int dp, const int64_t* off, int64_t N, const int32_t* mem_cl, const T* Y,        \
                             const T* x, const T* P, double* pm, int m, int d, int ld, cudaStream_t s) {       \
    ad2k::launch_cost_member_impl<T>(dp, off, N, mem_cl, Y, x, P, pm, m, d, ld, s);                             \
  }
