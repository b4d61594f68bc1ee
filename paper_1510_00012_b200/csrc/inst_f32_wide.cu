// inst_f32_wide.cu — launchers of the warp-pair iteration kernel (variant 3, 32 < m <= 64, fp32)
// and of the tiled cost build (ad2_wide.cuh).
#include <cstdlib>

#include "ad2_tc.cuh"
#include "ad2_wide.cuh"

namespace ad2k {

// (pairs per CTA, ring KB per pair): 0 = (2, 80) one CTA / SM with 4 warps; 1 = (3, 64) 6 warps;
// 2 = (4, 48) 8 warps (single-buffered: a ring that holds exactly one largest pass)
template <int NPAIR, int RKB, int DP>
static void go_wide(int mode, const IterArgs<float>& a, int64_t n_items, cudaStream_t s) {
  using Lay = WideLayout<NPAIR, RKB>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_badmm_wide<NPAIR, RKB, P1ONLY, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_wide<NPAIR, RKB, FUSED, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_wide<NPAIR, RKB, P2ONLY, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    attr = true;
  }
  dim3 g((unsigned)n_items), b(NPAIR * 64);
  if (mode == P1ONLY) k_badmm_wide<NPAIR, RKB, P1ONLY, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == FUSED) k_badmm_wide<NPAIR, RKB, FUSED, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else k_badmm_wide<NPAIR, RKB, P2ONLY, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
}

}  // namespace ad2k

using namespace ad2k;

int wide_cfg() {
  const char* e = getenv("AD2_WIDE_CFG");
  return (e && e[0] >= '0' && e[0] <= '2') ? e[0] - '0' : 2;
}
int wide_npair(int cfg) { return cfg == 1 ? 3 : cfg == 2 ? 4 : 2; }
size_t wide_cta_bytes(int cfg) {
  return cfg == 1 ? WideLayout<3, 64>::CTA_BYTES : cfg == 2 ? WideLayout<4, 48>::CTA_BYTES : WideLayout<2, 80>::CTA_BYTES;
}

template <int NPAIR, int RKB>
static void go_wide_d(int mode, int d, const IterArgs<float>& a, int64_t n_items, cudaStream_t s) {
  if (d <= 16) go_wide<NPAIR, RKB, 16>(mode, a, n_items, s);
  else go_wide<NPAIR, RKB, 64>(mode, a, n_items, s);
}

void launch_wide(int cfg, int mode, int d, const IterArgs<float>& a, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  if (cfg == 1) go_wide_d<3, 64>(mode, d, a, n_items, s);
  else if (cfg == 2) go_wide_d<4, 48>(mode, d, a, n_items, s);
  else go_wide_d<2, 80>(mode, d, a, n_items, s);
}

void launch_cost_tile(const int64_t* off, const int64_t* imb, const int32_t* icl, const float* Y, const float* x,
                      float* Cc, double* psum, int m, int d, int dy, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  if (d <= 16) k_cost_tile<16><<<(unsigned)n_items, 256, 0, s>>>(off, imb, icl, Y, x, Cc, psum, m, d, dy);
  else k_cost_tile<64><<<(unsigned)n_items, 256, 0, s>>>(off, imb, icl, Y, x, Cc, psum, m, d, dy);
}

void launch_cost_tc(const int64_t* off, const int64_t* imb, const int32_t* icl, const float* Y, const float* x,
                    float* Cc, double* psum, int m, int d, int dy, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  k_cost_tc<<<(unsigned)n_items, 128, 0, s>>>(off, imb, icl, Y, x, Cc, psum, m, d, dy);
}
