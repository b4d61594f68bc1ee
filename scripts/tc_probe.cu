// tc_probe.cu — standalone check of the per-warp tcgen05 cost contraction planned for the
// variant-2 iteration kernel (not part of the library):
//   A = x_c (32 centroid rows x 16 coords) split into tf32 hi / lo, written by every warp into
//       its own 32 TMEM lanes (tcgen05.st), so rows 32w + i of the M = 128 operand are x_i;
//   B = the warp's member points (N = 16 or 32 rows x 16 coords) split into hi / lo in the
//       canonical K-major no-swizzle layout (8-row core matrices of 16 B rows: LBO = K-chunk
//       stride 128 B, SBO = 8-row group stride 512 B);
//   D (TMEM columns 32w .. 32w + 31) = sum of the 4 split products over K = 16 (8 MMAs), read back
//       by the warp with tcgen05.ld 32x32b (lane i = row i).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tc_probe scripts/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>

__device__ __forceinline__ uint32_t sm32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                            // version
  return d;                                          // layout type 0: SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ float hi_tf32(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

// X [32][16], Y [4 warps][32 pts][16], out D [4][32 rows][32 cols]
__global__ void __launch_bounds__(128) k_probe(const float* X, const float* Y, float* D, int n_mma, int swap) {
  __shared__ __align__(128) float Bs[4][2][32 * 16];   // per warp: hi, lo (canonical layout)
  __shared__ uint32_t tm_d, tm_a;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sm32(&tm_d)));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sm32(&tm_a)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sm32(&bar[warp])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t td = tm_d, ta = tm_a;
  // A rows: lane i of every warp = x_i (hi in columns 0..15, lo in 16..31)
  {
    uint32_t r[32];
    for (int k = 0; k < 16; ++k) {
      const float v = X[lane * 16 + k];
      const float h = hi_tf32(v);
      r[k] = __float_as_uint(h);
      r[16 + k] = __float_as_uint(v - h);
    }
    const uint32_t a = ta + ((uint32_t)(32 * warp) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  // B: point j, chunk q (4 coords) -> (j/8)*512 + q*128 + (j%8)*16 bytes
  for (int it = lane; it < 32 * 4; it += 32) {
    const int j = it >> 2, q = it & 3;
    float4 v = *reinterpret_cast<const float4*>(Y + ((size_t)warp * 32 + j) * 16 + 4 * q);
    float4 h = make_float4(hi_tf32(v.x), hi_tf32(v.y), hi_tf32(v.z), hi_tf32(v.w));
    float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
    const int off = (j >> 3) * 128 + q * 32 + (j & 7) * 4;   // floats
    *reinterpret_cast<float4*>(&Bs[warp][0][off]) = h;
    *reinterpret_cast<float4*>(&Bs[warp][1][off]) = l;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t dcol = td + 32 * warp;
  if (lane == 0) {
    const uint32_t lbo = swap ? 512 : 128, sbo = swap ? 128 : 512;
    const uint32_t idesc = idesc_tf32(32);
    int first = 1;
    for (int term = 0; term < 4 && term < n_mma; ++term) {
      const int ah = (term == 2 || term == 3), bl = (term == 1 || term == 3);   // hh, hl, lh, ll
      for (int kq = 0; kq < 2; ++kq) {
        const uint64_t bd = desc_none(sm32(&Bs[warp][bl][kq * 64]), lbo, sbo);
        const uint32_t aa = ta + (ah ? 16 : 0) + 8 * kq;
        const uint32_t acc = first ? 0u : 1u;
        first = 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dcol),
            "r"(aa), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sm32(&bar[warp]))
                 : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred p;\nTW%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni TW%=;\n}" ::"r"(sm32(&bar[warp])), "r"(0)
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int h = 0; h < 8; ++h) {
    uint32_t r0, r1, r2, r3;
    const uint32_t a = td + ((uint32_t)(32 * warp) << 16) + 32 * warp + 4 * h;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float* o = D + ((size_t)warp * 32 + lane) * 32 + 4 * h;
    o[0] = __uint_as_float(r0); o[1] = __uint_as_float(r1); o[2] = __uint_as_float(r2); o[3] = __uint_as_float(r3);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(td));
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(ta));
  }
}

int main() {
  std::mt19937 g(1);
  std::normal_distribution<float> nd(0.f, 3.f);
  std::vector<float> X(32 * 16), Y(4 * 32 * 16), D(4 * 32 * 32);
  for (auto& v : X) v = nd(g);
  for (auto& v : Y) v = nd(g);
  float *dX, *dY, *dD;
  cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dY, Y.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  for (int swap = 0; swap < 2; ++swap)
    for (int terms : {1, 3, 4}) {
      cudaMemset(dD, 0, D.size() * 4);
      k_probe<<<1, 128>>>(dX, dY, dD, terms, swap);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("swap %d terms %d: %s\n", swap, terms, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double maxrel = 0, maxabs = 0;
      for (int w = 0; w < 4; ++w)
        for (int i = 0; i < 32; ++i)
          for (int j = 0; j < 32; ++j) {
            double s = 0, sa = 0;
            for (int k = 0; k < 16; ++k) {
              s += (double)X[i * 16 + k] * Y[(w * 32 + j) * 16 + k];
              sa += fabs((double)X[i * 16 + k] * Y[(w * 32 + j) * 16 + k]);
            }
            const double err = fabs(D[(w * 32 + i) * 32 + j] - s);
            maxabs = fmax(maxabs, err);
            maxrel = fmax(maxrel, err / sa);
          }
      printf("swap %d terms %d: max |err| %.3e, max |err| / sum|x_k y_k| %.3e (2^-22 = %.2e, 2^-24 = %.2e)\n", swap,
             terms, maxabs, maxrel, ldexp(1.0, -22), ldexp(1.0, -24));
    }
  return 0;
}
