// inst_f64_mp8.cu — explicit instantiations of the fused B-ADMM iteration kernels for
// T=double, MP=8 (split per (dtype, MP) so nvcc compiles the template set in parallel).
//   variant 2: k_badmm_tma  (TMA-staged, cost recomputed; ad2_tma.cuh)
#include "ad2_tma.cuh"

namespace ad2k {

template <int NCH, int DP>
static void go_tma(int mode, const IterArgs<double>& a, int64_t n_items, cudaStream_t s) {
  using Lay = TmaLayout<double, 8, NCH, DP>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_badmm_tma<double, 8, NCH, P1ONLY, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<double, 8, NCH, FUSED, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<double, 8, NCH, P2ONLY, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<double, 8, NCH, P1INIT, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<double, 8, NCH, P2X, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_tma<double, 8, NCH, FUSEDX, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    attr = true;
  }
  dim3 g((unsigned)n_items), b(NWARP * 32);
  if (mode == P1ONLY) k_badmm_tma<double, 8, NCH, P1ONLY, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == FUSED) k_badmm_tma<double, 8, NCH, FUSED, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == P1INIT) k_badmm_tma<double, 8, NCH, P1INIT, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == P2X) k_badmm_tma<double, 8, NCH, P2X, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == FUSEDX) k_badmm_tma<double, 8, NCH, FUSEDX, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else k_badmm_tma<double, 8, NCH, P2ONLY, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
}

template <int NCH>
static void go_nch(int variant, int mode, int dp, const IterArgs<double>& a, int64_t n_items, cudaStream_t s) {
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
size_t tma_cta_bytes<double, 8>(int nch, int dp) {
  auto f = [](size_t a, size_t b) { return a + b; };
  if (nch == 2 && 8 < 32) {
    if (dp <= 4) return f(TmaLayout<double, 8, (8 < 32 ? 2 : 1), 4>::CTA_BYTES, TmaLayout<double, 8, (8 < 32 ? 2 : 1), 4>::STATIC_BYTES);
    return f(TmaLayout<double, 8, (8 < 32 ? 2 : 1), 16>::CTA_BYTES, TmaLayout<double, 8, (8 < 32 ? 2 : 1), 16>::STATIC_BYTES);
  }
  if (dp <= 4) return f(TmaLayout<double, 8, 1, 4>::CTA_BYTES, TmaLayout<double, 8, 1, 4>::STATIC_BYTES);
  return f(TmaLayout<double, 8, 1, 16>::CTA_BYTES, TmaLayout<double, 8, 1, 16>::STATIC_BYTES);
}

template <typename T, int MP>
void launch_warp(int variant, int mode, int nch, int dp, const IterArgs<T>& a, int64_t n_items, cudaStream_t s);

template <>
void launch_warp<double, 8>(int variant, int mode, int nch, int dp, const IterArgs<double>& a, int64_t n_items,
                           cudaStream_t s) {
  if (nch == 2) go_nch<2>(variant, mode, dp, a, n_items, s);
  else go_nch<1>(variant, mode, dp, a, n_items, s);
}
