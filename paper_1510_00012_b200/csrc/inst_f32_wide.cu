// inst_f32_wide.cu — launchers of the warp-pair iteration kernel (variant 3, 32 < m <= 64, fp32)
// and of the tiled cost build (ad2_wide.cuh).
#include <cstdlib>

#include "ad2_launch.cuh"
#include "ad2_tc.cuh"
#include "ad2_wide.cuh"

namespace ad2k {

// instantiations (rows per member WM, largest m_k MKX, groups per CTA, ring KB per group):
//   (32, 64, 8, 24) (64, 64, 4, 48) (128, 64, 2, 96) (32, 128, 4, 48) (64, 128, 2, 96) (128, 128, 1, 192)
template <int WM, int MKX, int NPAIR, int RKB, int DP>
static void go_wide(int mode, const IterArgs<float>& a, int64_t n_items, cudaStream_t s) {
  using Lay = WideLayout<WM, MKX, NPAIR, RKB>;
  static PerDevice once;                   // the smem attribute is per device
  if (once.first()) {
    cudaFuncSetAttribute(k_badmm_wide<WM, MKX, NPAIR, RKB, P1ONLY, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_wide<WM, MKX, NPAIR, RKB, FUSED, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_wide<WM, MKX, NPAIR, RKB, P2ONLY, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_wide<WM, MKX, NPAIR, RKB, P2X, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_wide<WM, MKX, NPAIR, RKB, FUSEDX, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    cudaFuncSetAttribute(k_badmm_wide<WM, MKX, NPAIR, RKB, P1INIT, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::CTA_BYTES);
    once.done();
  }
  dim3 g((unsigned)n_items), b(NPAIR * WM);
  if (mode == P1ONLY) k_badmm_wide<WM, MKX, NPAIR, RKB, P1ONLY, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == FUSED) k_badmm_wide<WM, MKX, NPAIR, RKB, FUSED, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == P2X) k_badmm_wide<WM, MKX, NPAIR, RKB, P2X, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == FUSEDX) k_badmm_wide<WM, MKX, NPAIR, RKB, FUSEDX, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else if (mode == P1INIT) k_badmm_wide<WM, MKX, NPAIR, RKB, P1INIT, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
  else k_badmm_wide<WM, MKX, NPAIR, RKB, P2ONLY, DP><<<g, b, Lay::CTA_BYTES, s>>>(a);
}

template <int WM, int MKX, int NPAIR, int RKB>
static void go_wide_d(int mode, int d, const IterArgs<float>& a, int64_t n_items, cudaStream_t s) {
  if (d <= 16) go_wide<WM, MKX, NPAIR, RKB, 16>(mode, a, n_items, s);
  else go_wide<WM, MKX, NPAIR, RKB, 64>(mode, a, n_items, s);
}

}  // namespace ad2k

using namespace ad2k;

// kernel configuration id: wm (32 / 64 / 128) + (mkx == 128 ? 1 : 0)
int wide_npair(int cfg) {
  const int wm = cfg & ~1, big = cfg & 1;
  if (!big) return wm == 32 ? 8 : wm == 64 ? 4 : 2;
  return wm == 32 ? 4 : wm == 64 ? 2 : 1;
}
size_t wide_cta_bytes(int cfg) {
  switch (cfg) {
    case 32: return WideLayout<32, 64, 8, 24>::CTA_BYTES;
    case 64: return WideLayout<64, 64, 4, 48>::CTA_BYTES;
    case 128: return WideLayout<128, 64, 2, 96>::CTA_BYTES;
    case 33: return WideLayout<32, 128, 4, 48>::CTA_BYTES;
    case 65: return WideLayout<64, 128, 2, 96>::CTA_BYTES;
    default: return WideLayout<128, 128, 1, 192>::CTA_BYTES;
  }
}

void launch_wide(int cfg, int mode, int d, const IterArgs<float>& a, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  switch (cfg) {
    case 32: go_wide_d<32, 64, 8, 24>(mode, d, a, n_items, s); break;
    case 64: go_wide_d<64, 64, 4, 48>(mode, d, a, n_items, s); break;
    case 128: go_wide_d<128, 64, 2, 96>(mode, d, a, n_items, s); break;
    case 33: go_wide_d<32, 128, 4, 48>(mode, d, a, n_items, s); break;
    case 65: go_wide_d<64, 128, 2, 96>(mode, d, a, n_items, s); break;
    default: go_wide_d<128, 128, 1, 192>(mode, d, a, n_items, s); break;
  }
}

void launch_cost_tile(const int64_t* off, const int64_t* imb, const int32_t* icl, const float* Y, const float* x,
                      float* Cc, double* psum, int m, int d, int dy, int ld, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  static PerDevice once;                   // the smem attribute is per device
  if (once.first()) {
    cudaFuncSetAttribute(k_cost_tile<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CostTile<16>::BYTES);
    cudaFuncSetAttribute(k_cost_tile<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CostTile<64>::BYTES);
    once.done();
  }
  static const bool tile4 = getenv("AD2_COST_TILE4") != nullptr;   // A/B knob: the 4 x 4 thread tiles
  if (d > 16 && !tile4) {
    static PerDevice once8;
    if (once8.first()) {
      cudaFuncSetAttribute(k_cost_tile8, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CostTile8::BYTES);
      once8.done();
    }
    k_cost_tile8<<<(unsigned)n_items, 128, CostTile8::BYTES, s>>>(off, imb, icl, Y, x, Cc, psum, m, d, dy, ld);
    return;
  }
  if (d <= 16)
    k_cost_tile<16><<<(unsigned)n_items, 256, CostTile<16>::BYTES, s>>>(off, imb, icl, Y, x, Cc, psum, m, d, dy, ld);
  else
    k_cost_tile<64><<<(unsigned)n_items, 256, CostTile<64>::BYTES, s>>>(off, imb, icl, Y, x, Cc, psum, m, d, dy, ld);
}

void launch_cost_tc(const int64_t* off, const int64_t* imb, const int32_t* icl, const float* Y, const float* x,
                    float* Cc, double* psum, int m, int d, int dy, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  k_cost_tc<<<(unsigned)n_items, 128, 0, s>>>(off, imb, icl, Y, x, Cc, psum, m, d, dy);
}

// fp32-accurate 3 x TF32 tensor-core cost build (ld 64)
void launch_cost_tc32(const int64_t* off, const int64_t* imb, const int32_t* icl, const float* Y, const float* x,
                      double* ct, int K, float* Cc, double* psum, int m, int d, int dy, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  k_cost_centre<<<K, 64, 0, s>>>(x, ct, m, d);
  constexpr int SMEM = 98304 + 1024;             // + alignment slack
  static PerDevice once;
  if (once.first()) {
    cudaFuncSetAttribute(k_cost_tc32, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    once.done();
  }
  k_cost_tc32<<<(unsigned)n_items, 128, SMEM, s>>>(off, imb, icl, Y, x, ct, Cc, psum, m, d, dy);
}

void launch_cost_tile_big(const int64_t* off, const int64_t* imb, const int32_t* icl, const float* Y, const float* x,
                          float* Cc, double* psum, int m, int d, int dy, int ld, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  k_cost_tile_big<<<(unsigned)n_items, 256, 0, s>>>(off, imb, icl, Y, x, Cc, psum, m, d, dy, ld);
}

void launch_xpart(const int64_t* off, const int64_t* imb, const float* Q, const float* Y, float* px, int m, int d,
                  int dy, int ld, int parts, int64_t n_items, cudaStream_t s) {
  if (n_items == 0) return;
  k_xpart<<<(unsigned)n_items, 256, 0, s>>>(off, imb, Q, Y, px, m, d, dy, ld, parts);
}
