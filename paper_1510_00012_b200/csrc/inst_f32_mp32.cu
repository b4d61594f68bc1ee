// inst_f32_mp32.cu — explicit instantiations of the fused B-ADMM iteration kernels for
// T=float, MP=32 (split per (dtype, MP) so nvcc compiles the template set in parallel).
//   variant 2: k_badmm_tma  (TMA-staged, cost recomputed; ad2_tma.cuh)
#include "ad2_tma.cuh"

namespace ad2k {

template <int NCH, int DP>
static void go_tma(int mode, const IterArgs<float>& a, int64_t n_items, cudaStream_t s) {
  using Lay = TmaLayout<float, 32, NCH, DP>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_badmm_tma<float, 32, NCH, P1ONLY, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<float, 32, NCH, FUSED, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<float, 32, NCH, P2ONLY, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<float, 32, NCH, P1INIT, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<float, 32, NCH, P2X, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<float, 32, NCH, FUSEDX, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    attr = true;
  }
  dim3 g((unsigned)n_items), b(NWARP * 32);
  if (mode == P1ONLY) k_badmm_tma<float, 32, NCH, P1ONLY, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == FUSED) k_badmm_tma<float, 32, NCH, FUSED, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == P1INIT) k_badmm_tma<float, 32, NCH, P1INIT, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == P2X) k_badmm_tma<float, 32, NCH, P2X, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == FUSEDX) k_badmm_tma<float, 32, NCH, FUSEDX, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else k_badmm_tma<float, 32, NCH, P2ONLY, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
}

template <int NCH>
static void go_nch(int variant, int mode, int dp, const IterArgs<float>& a, int64_t n_items, cudaStream_t s) {
  if (variant == 2) {
    if (dp <= 4) go_tma<NCH, 4>(mode, a, n_items, s);
    else go_tma<NCH, 16>(mode, a, n_items, s);
  }
}

}  // namespace ad2k

using namespace ad2k;

template <typename T, int MP>
size_t tma_cta_bytes(int nch, int dp);

template <>
size_t tma_cta_bytes<float, 32>(int nch, int dp) {
  auto f = [](size_t a, size_t b) { return a + b; };
  if (nch == 2 && 32 < 32) {
    if (dp <= 4) return f(TmaLayout<float, 32, (32 < 32 ? 2 : 1), 4>::CTA_BYTES, TmaLayout<float, 32, (32 < 32 ? 2 : 1), 4>::STATIC_BYTES);
    return f(TmaLayout<float, 32, (32 < 32 ? 2 : 1), 16>::CTA_BYTES, TmaLayout<float, 32, (32 < 32 ? 2 : 1), 16>::STATIC_BYTES);
  }
  if (dp <= 4) return f(TmaLayout<float, 32, 1, 4>::CTA_BYTES, TmaLayout<float, 32, 1, 4>::STATIC_BYTES);
  return f(TmaLayout<float, 32, 1, 16>::CTA_BYTES, TmaLayout<float, 32, 1, 16>::STATIC_BYTES);
}

template <typename T, int MP>
void launch_warp(int variant, int mode, int nch, int dp, const IterArgs<T>& a, int64_t n_items, cudaStream_t s);

template <>
void launch_warp<float, 32>(int variant, int mode, int nch, int dp, const IterArgs<float>& a, int64_t n_items,
                           cudaStream_t s) {
  (void)nch;
  go_nch<1>(variant, mode, dp, a, n_items, s);
}

template <typename T>
void launch_cost_member(int dp, const int64_t* off, int64_t N, const int32_t* mem_cl, const T* Y, const T* x,
                        const T* P, double* pm, int m, int d, int ld, cudaStream_t s);

template <>
void launch_cost_member<float>(int dp, const int64_t* off, int64_t N, const int32_t* mem_cl, const float* Y,
                             const float* x, const float* P, double* pm, int m, int d, int ld, cudaStream_t s) {
  if (N == 0) return;
  constexpr int NW = cost_member_warps<float>();
  static int grid_cap = 0;                             // resident CTAs (grid-stride kernel)
  if (!grid_cap) {
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cost_member<float, 16>, 32 * NW, 0);
    grid_cap = nsm * (per > 0 ? per : 1);
  }
  const int64_t need = (N + NW - 1) / NW;
  const unsigned g = (unsigned)(need < grid_cap ? need : grid_cap);
  if (dp <= 4) k_cost_member<float, 4><<<g, 32 * NW, 0, s>>>(off, N, mem_cl, Y, x, P, pm, m, d, ld);
  else k_cost_member<float, 16><<<g, 32 * NW, 0, s>>>(off, N, mem_cl, Y, x, P, pm, m, d, ld);
}
