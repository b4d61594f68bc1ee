// inst_f64_mp8.cu — explicit instantiations of the fused B-ADMM kernel for T=double, MP=8
// (split so nvcc compiles the template set in parallel).  See ad2_kernels.cuh.
#include "ad2_kernels.cuh"

namespace ad2k {

template <int NCH, int DP>
static void go(int mode, const IterArgs<double>& a, int64_t n_items, cudaStream_t s) {
  dim3 g((unsigned)n_items), b(NWARP * 32);
  if (mode == P1ONLY) k_badmm_warp<double, 8, NCH, P1ONLY, 1><<<g, b, 0, s>>>(a);
  else if (mode == FUSED) k_badmm_warp<double, 8, NCH, FUSED, 1><<<g, b, 0, s>>>(a);
  else k_badmm_warp<double, 8, NCH, P2ONLY, DP><<<g, b, 0, s>>>(a);
}

template <int NCH>
static void go_dp(int mode, int dp, const IterArgs<double>& a, int64_t n_items, cudaStream_t s) {
  if (dp <= 4) go<NCH, 4>(mode, a, n_items, s);
  else go<NCH, 16>(mode, a, n_items, s);

}

}  // namespace ad2k

using namespace ad2k;

template <typename T, int MP>
void launch_warp(int mode, int nch, int dp, const IterArgs<T>& a, int64_t n_items, cudaStream_t s);

template <>
void launch_warp<double, 8>(int mode, int nch, int dp, const IterArgs<double>& a, int64_t n_items, cudaStream_t s) {
  if (nch == 2) go_dp<2>(mode, dp, a, n_items, s);
  else go_dp<1>(mode, dp, a, n_items, s);
}
