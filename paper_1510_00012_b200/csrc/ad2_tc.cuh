// ad2_tc.cuh — tensor-core (tcgen05, bf16 in / fp32 accumulate in TMEM) cost build for the
// cached-cost kernels (d = 64, where C is a dense contraction).
//
//   C_ij = |x_i|^2 + |y_j|^2 - 2 x_i . y_j     (squared Euclidean ground distance)
//
// For cluster c the points of a work item are contiguous, and the cost blocks of its members
// (column-major m x m_k, ld = 64) are one contiguous point-major array: C[(p0 + p) * 64 + i].
// One CTA (4 warps) per work item; per tile of 128 points:
//   A = Y tile (M = 128 points x K = 64 coords, bf16, K-major, 128-byte swizzle), converted from
//       the fp32 supports by all threads (|y_p|^2 kept in fp32),
//   B = x_c (N = 64 centroid rows x K = 64, bf16, K-major, 128-byte swizzle), staged once,
//   D = A B^T in TMEM (128 lanes = points x 64 fp32 columns = centroid rows), 4 MMAs of K = 16,
// then each thread reads its point's 64 accumulators (tcgen05.ld 32x32b) and writes the 64
// costs (256 contiguous bytes) with |x_i|^2 and |y_p|^2 added in fp32 and the result clamped
// at 0.  bf16 operands bound the error by |dC| <= 2^-7 |x_i| |y_j| (+ fp32 rounding): this one
// is params->cost_mode = 1; the parity default is the fp32 FFMA2 tile build (k_cost_tile).
#pragma once
#include <cuda_bf16.h>

#include "ad2_kernels.cuh"

namespace ad2k {

__device__ __forceinline__ uint32_t tc_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// shared-memory matrix descriptor (sm_100 UMMA): K-major, 128-byte swizzle, 8-row atoms of
// 1024 bytes (stride byte offset), version 1
__device__ __forceinline__ uint64_t tc_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);            // start address
  d |= (uint64_t)1 << 16;                            // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                  // stride byte offset: next 8-row atom
  d |= (uint64_t)1 << 46;                            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
  return d;
}

// instruction descriptor, kind::f16: D fp32, A/B bf16, both K-major, N = 64, M = 128
constexpr uint32_t TC_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

// byte offset of element (row r, k) in a K-major 128B-swizzled tile with 64 bf16 per row
__device__ __forceinline__ uint32_t tc_sw128_off(int r, int k) {
  const int chunk = (k >> 3) ^ (r & 7);              // 16-byte chunk, XOR-swizzled by the row
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + chunk * 16 + (k & 7) * 2);
}

__global__ void __launch_bounds__(128)
k_cost_tc(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
          const int32_t* __restrict__ item_cl, const float* __restrict__ Y, const float* __restrict__ x,
          float* __restrict__ Cc, double* __restrict__ psum, int m, int d, int dy) {
  __shared__ __align__(1024) unsigned char sA[128 * 128];     // 16 KB, 16 atoms
  __shared__ __align__(1024) unsigned char sB[64 * 128];      // 8 KB
  __shared__ __align__(16) float4 sO[4][32][8];                // per warp: 32 points x 32 costs (16 KB)
  __shared__ float xx[64], yy[128];
  __shared__ uint32_t tmem_base_s;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ double red[4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int item = blockIdx.x;
  const int c = item_cl[item];

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(tc_smem(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // B = x_c in bf16 (rows >= m and coordinates >= d are zero), |x_i|^2 in fp32
  for (int v = tid; v < 64 * 8; v += 128) {            // (row, 8-coordinate chunk)
    const int r = v >> 3, k0 = (v & 7) * 8;
    __align__(16) __nv_bfloat16 h[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u;
      h[u] = __float2bfloat16_rn((r < m && k < d) ? x[((int64_t)c * m + r) * d + k] : 0.f);
    }
    *reinterpret_cast<uint4*>(sB + tc_sw128_off(r, k0)) = *reinterpret_cast<const uint4*>(h);
  }
  if (tid < 64) {
    float s = 0.f;
    for (int k = 0; k < d; ++k) {
      const float v = tid < m ? x[((int64_t)c * m + tid) * d + k] : 0.f;
      s = fmaf(v, v, s);
    }
    xx[tid] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  const int64_t p_beg = off[item_mb[item]], p_end = off[item_mb[item + 1]];
  double acc = 0.0;
  uint32_t phase = 0;
  // the Y tile in fp32 registers: 16 threads per point row, 4 coordinates each (coalesced reads),
  // all 16 loads of a thread issued before the first is consumed (memory-level parallelism; loading
  // the next tile during the MMA and epilogue instead needs 156 registers, 3 CTAs per SM: slower)
  float4 fv[16];
  auto load_tile = [&](int64_t t0) {
    const int n = (int)((p_end - t0) < 128 ? (p_end - t0) : 128);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int v = tid + 128 * u;
      const int r = v >> 4, k0 = (v & 15) * 4;
      fv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < n && k0 < d) fv[u] = *reinterpret_cast<const float4*>(Y + (t0 + r) * dy + k0);   // dy % 4 == 0, pad = 0
    }
  };
  for (int64_t q0 = p_beg; q0 < p_end; q0 += 128) {
    const int np = (int)((p_end - q0) < 128 ? (p_end - q0) : 128);
    load_tile(q0);
    // A = Y tile in bf16
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int v = tid + 128 * u;
      const int r = v >> 4, k0 = (v & 15) * 4;
      const float4 f = fv[u];
      float s = f.x * f.x + f.y * f.y + f.z * f.z + f.w * f.w;
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((v & 15) == 0) yy[r] = s;
      __align__(8) __nv_bfloat16 h[4] = {__float2bfloat16_rn(f.x), __float2bfloat16_rn(f.y),
                                         __float2bfloat16_rn(f.z), __float2bfloat16_rn(f.w)};
      *reinterpret_cast<uint2*>(sA + tc_sw128_off(r, k0)) = *reinterpret_cast<const uint2*>(h);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t da = tc_desc_sw128(tc_smem(sA)), db = tc_desc_sw128(tc_smem(sB));
#pragma unroll
      for (int k = 0; k < 4; ++k) {                    // K = 16 per MMA: +32 bytes in the swizzle atom
        const uint64_t a_k = da + (uint64_t)(2 * k), b_k = db + (uint64_t)(2 * k);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(a_k), "l"(b_k), "r"(TC_IDESC), "r"(k));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       tc_smem(&mbar))
                   : "memory");
    }
    // wait for the accumulator
    asm volatile(
        "{\n\t.reg .pred p;\nTW%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra.uni TW%=;\n}" ::"r"(tc_smem(&mbar)),
        "r"(phase)
        : "memory");
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: thread (warp, lane) = point 32 warp + lane; TMEM lanes 32 warp .. 32 warp + 31
    const int p = 32 * warp + lane;
    const float yp = yy[p];
    float s = 0.f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t r[32];
      const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(32 * h);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
            "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
            "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
            "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // the point's 32 costs of this half into the warp's tile (16-byte chunk u at u ^ (p & 7):
      // conflict-free), then the warp stores 4 points' 128-byte half rows per instruction
      if (p < np) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 32 * h + 4 * u + e;
            const float dot = __uint_as_float(r[4 * u + e]);
            o[e] = (i < m) ? fmaxf(fmaf(-2.f, dot, xx[i] + yp), 0.f) : 0.f;
            s += o[e];
          }
          sO[warp][lane][u ^ (lane & 7)] = make_float4(o[0], o[1], o[2], o[3]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int pl = 4 * k + (lane >> 3), u = lane & 7;     // point within the warp, chunk
        if (32 * warp + pl < np)
          reinterpret_cast<float4*>(Cc + (q0 + 32 * warp + pl) * 64 + 32 * h)[u] = sO[warp][pl][u ^ (pl & 7)];
      }
      __syncwarp();
    }
    acc += (double)s;
    // TMEM and the A tile are reused by the next tile
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
  }
  if (psum) {
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid == 0) psum[item] = (red[0] + red[1]) + (red[2] + red[3]);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

}  // namespace ad2k

namespace ad2k {

// ---------------------------------------------------------------------------------------------
// fp32-accurate tensor-core cost build: 3 x TF32 (tcgen05.mma kind::tf32).  The points are
// centred on the cluster's mean centroid point o (k_cost_centre; C is translation invariant), each
// operand is split into hi = tf32(v) and lo = tf32(v - hi) (11 + 11 significant bits), and
//   x'.y' = x'_hi.y'_hi + x'_hi.y'_lo + x'_lo.y'_hi   (+ x'_lo.y'_lo, ~2^-22 relative, dropped)
// is accumulated in fp32 in TMEM: 24 MMAs (3 terms x K = 64 in steps of 8) per 128-point tile;
// C = |x'|^2 + |y'|^2 - 2 x'.y'.  The rho numerator (psum) is the closed form
// sum_p (m |y'_p|^2 - 2 S.y'_p) + X2 in fp64 with exact operands, not a sum of the built C.
// Operands are K-major with the 128-byte swizzle: a 64-element fp32 row spans two 128-byte
// K-blocks, stored as two [rows][128 B] tiles.  Opt-in (AD2_COST_TC32=1): uncentred, the
// accumulation's ~2^-20 relative error on |x||y| broke the 1e-5 plan parity on config 4's unit
// vectors (round 1); centred with the closed-form rho, the whole GPU suite passes on it, but the
// single-stage pipeline (2 CTAs per SM, loads -> MMA -> epilogue in sequence) took 8.7 ms on
// config 4; with the next tile's rows loaded into registers during the MMAs and the epilogue the
// config-4 round is the same as with the FFMA2 tile build (317.7 vs 318.6 ms).
// ---------------------------------------------------------------------------------------------
// instruction descriptor, kind::tf32: D fp32, A/B tf32 (format 2), K-major, N = 64, M = 128
constexpr uint32_t TC32_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

// byte offset of fp32 element (row r, k) in a tile of R rows x 64 k: K-block kb = k / 32 of
// R x 128 bytes, 8-row swizzle atoms of 1024 bytes, 16-byte chunks XOR-swizzled by the row
__device__ __forceinline__ uint32_t tc32_off(int R, int r, int k) {
  const int kb = k >> 5, kin = k & 31;
  const int chunk = (kin >> 2) ^ (r & 7);
  return (uint32_t)(kb * R * 128 + (r >> 3) * 1024 + (r & 7) * 128 + chunk * 16 + (kin & 3) * 4);
}

__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(v));
  return __uint_as_float(u);
}

// Per-cluster centre for the 3 x TF32 build (one CTA of 64 threads per cluster c, d <= 64):
//   o_c = mean of the m centroid points (fp32), S_k = sum_i (x_ik - o_k) and
//   X2 = sum_i |x_i - o|^2 in fp64 (exact operands: fp32 differences are exact in fp64), and
//   xx_i = |x_i - o|^2 in fp32 for the epilogue.  Layout of ct per cluster (CT_WORDS doubles):
//   [o: 64 floats = 32 doubles | xx: 64 floats = 32 doubles | S: 64 doubles | X2: 1 double | pad]
//   (CT_WORDS, ad2_kernels.cuh)
__global__ void __launch_bounds__(64) k_cost_centre(const float* __restrict__ x, double* __restrict__ ct, int m, int d) {
  const int c = blockIdx.x, k = threadIdx.x;
  double* cc = ct + (size_t)c * CT_WORDS;
  float* o = reinterpret_cast<float*>(cc);
  float* xx = reinterpret_cast<float*>(cc + 32);
  __shared__ float os[64];
  __shared__ double x2s[64];
  float ok = 0.f;
  double s1 = 0.0, s2 = 0.0;
  if (k < d) {
    double sm = 0.0;
    for (int i = 0; i < m; ++i) sm += (double)x[((int64_t)c * m + i) * d + k];
    ok = (float)(sm / m);
    for (int i = 0; i < m; ++i) {
      const double v = (double)x[((int64_t)c * m + i) * d + k] - (double)ok;
      s1 += v;
      s2 = fma(v, v, s2);
    }
  }
  os[k] = ok;
  x2s[k] = s2;
  o[k] = ok;
  cc[64 + k] = s1;
  __syncthreads();
  if (k == 0) {
    double t = 0.0;
    for (int j = 0; j < 64; ++j) t += x2s[j];
    cc[128] = t;
  }
  float sx = 0.f;                                     // row k: |x_k - o|^2 in fp32
  if (k < m)
    for (int j = 0; j < d; ++j) {
      const float v = x[((int64_t)c * m + k) * d + j] - os[j];
      sx = fmaf(v, v, sx);
    }
  xx[k] = sx;
}

__global__ void __launch_bounds__(128)
k_cost_tc32(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
            const int32_t* __restrict__ item_cl, const float* __restrict__ Y, const float* __restrict__ x,
            const double* __restrict__ ct, float* __restrict__ Cc, double* __restrict__ psum, int m, int d, int dy) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  // the 128-byte swizzle needs 1024-byte aligned atoms: align the dynamic region by hand
  unsigned char* tsm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(tsm_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* sAh = tsm;                          // 128 x 64 fp32 = 32 KB each
  unsigned char* sAl = tsm + 32768;
  unsigned char* sBh = tsm + 65536;                  // 64 x 64 fp32 = 16 KB each
  unsigned char* sBl = tsm + 81920;
  __shared__ float xx[64], yy[128], oc[64];
  __shared__ double sxd[64], x2d[64];
  __shared__ uint32_t tmem_base_s;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ double red[4];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int item = blockIdx.x;
  const int c = item_cl[item];

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(tc_smem(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the cluster's centre and fp64 sums (k_cost_centre)
  {
    const double* cc = ct + (size_t)c * CT_WORDS;
    if (tid < 64) {
      oc[tid] = reinterpret_cast<const float*>(cc)[tid];
      xx[tid] = reinterpret_cast<const float*>(cc + 32)[tid];
      sxd[tid] = cc[64 + tid];
    }
    if (tid == 0) x2d[0] = cc[128];
  }
  __syncthreads();
  // B = x'_c split into tf32 hi / lo (rows >= m and coordinates >= d are zero); |x'_i|^2 in fp32
  for (int v = tid; v < 64 * 16; v += 128) {
    const int r = v >> 4, k0 = (v & 15) * 4;
    float4 h, l;
    float* he = reinterpret_cast<float*>(&h);
    float* le = reinterpret_cast<float*>(&l);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float val = (r < m && k0 + u < d) ? x[((int64_t)c * m + r) * d + k0 + u] - oc[k0 + u] : 0.f;
      he[u] = tf32_rna(val);
      le[u] = tf32_rna(val - he[u]);
    }
    *reinterpret_cast<float4*>(sBh + tc32_off(64, r, k0)) = h;
    *reinterpret_cast<float4*>(sBl + tc32_off(64, r, k0)) = l;
  }
  const double x2tot = x2d[0];                        // sum_i |x_i - o|^2 (fp64)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  const int64_t p_beg = off[item_mb[item]], p_end = off[item_mb[item + 1]];
  double acc = 0.0;
  uint32_t phase = 0;
  // thread tid converts coordinates k0 .. k0+3 of tile rows tid/16 + 8 it (it < 16); the next
  // tile's rows are loaded into registers while this tile's MMAs and epilogue run
  const int kq = (tid & 15) * 4, rq = tid >> 4;
  float4 yr[16];
  auto load_tile = [&](int64_t qs) {
    const int npn = (int)((p_end - qs) < 128 ? (p_end - qs) : 128);
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int r = rq + 8 * it;
      yr[it] = (r < npn && kq < d) ? __ldg(reinterpret_cast<const float4*>(Y + (qs + r) * dy + kq))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);   // dy % 4 == 0
    }
  };
  if (p_beg < p_end) load_tile(p_beg);
  for (int64_t q0 = p_beg; q0 < p_end; q0 += 128) {
    const int np = (int)((p_end - q0) < 128 ? (p_end - q0) : 128);
    // A = Y' tile split into tf32 hi / lo: 16 threads per point row, 4 coordinates each
#pragma unroll
    for (int it = 0; it < 16; ++it) {
      const int r = rq + 8 * it, k0 = kq;
      float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
      double q = 0.0;                                  // this chunk's part of sum_i |x_i - y_p|^2
      if (r < np && k0 < d) {
        const float4 y4 = yr[it];
        const float* ye = reinterpret_cast<const float*>(&y4);
        float* fe = reinterpret_cast<float*>(&f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (k0 + u < d) {
            fe[u] = ye[u] - oc[k0 + u];
            if (psum) {                                // fp64: m (y - o)^2 - 2 S_k (y - o), exact operands
              const double yd = (double)ye[u] - (double)oc[k0 + u];
              q = fma(yd, (double)m * yd - 2.0 * sxd[k0 + u], q);
            }
          }
        }
      }
      float s = fmaf(f.x, f.x, fmaf(f.y, f.y, fmaf(f.z, f.z, f.w * f.w)));
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((tid & 15) == 0) yy[r] = s;
      if (psum) {
#pragma unroll
        for (int o = 8; o >= 1; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        if ((tid & 15) == 0 && r < np) acc += q + x2tot;   // rho numerator in closed form (fp64)
      }
      const float4 h = make_float4(tf32_rna(f.x), tf32_rna(f.y), tf32_rna(f.z), tf32_rna(f.w));
      const float4 l = make_float4(tf32_rna(f.x - h.x), tf32_rna(f.y - h.y), tf32_rna(f.z - h.z), tf32_rna(f.w - h.w));
      *reinterpret_cast<float4*>(sAh + tc32_off(128, r, k0)) = h;
      *reinterpret_cast<float4*>(sAl + tc32_off(128, r, k0)) = l;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned char* As[3] = {sAh, sAh, sAl};
      const unsigned char* Bs[3] = {sBh, sBl, sBh};
      int first = 1;
#pragma unroll
      for (int term = 0; term < 3; ++term) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {             // K = 8 tf32 (32 bytes) per MMA
          const int kb = kk >> 2, kin = kk & 3;
          const uint64_t da = tc_desc_sw128(tc_smem(As[term] + kb * 128 * 128)) + (uint64_t)(2 * kin);
          const uint64_t db = tc_desc_sw128(tc_smem(Bs[term] + kb * 64 * 128)) + (uint64_t)(2 * kin);
          const uint32_t accum = first ? 0u : 1u;
          first = 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(da), "l"(db), "r"(TC32_IDESC), "r"(accum));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       tc_smem(&mbar))
                   : "memory");
    }
    if (q0 + 128 < p_end) load_tile(q0 + 128);       // in flight during the MMAs and the epilogue
    asm volatile(
        "{\n\t.reg .pred p;\nTW%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra.uni TW%=;\n}" ::"r"(tc_smem(&mbar)),
        "r"(phase)
        : "memory");
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int p = 32 * warp + lane;
    const float yp = yy[p];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t r[32];
      const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(32 * h);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
            "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
            "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
            "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (p < np) {
        float4* dst = reinterpret_cast<float4*>(Cc + (q0 + p) * 64 + 32 * h);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          float o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 32 * h + 4 * u + e;
            const float dot = __uint_as_float(r[4 * u + e]);
            o[e] = (i < m) ? fmaxf(fmaf(-2.f, dot, xx[i] + yp), 0.f) : 0.f;
          }
          dst[u] = make_float4(o[0], o[1], o[2], o[3]);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
  }
  if (psum) {
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid == 0) psum[item] = (red[0] + red[1]) + (red[2] + red[3]);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

}  // namespace ad2k
