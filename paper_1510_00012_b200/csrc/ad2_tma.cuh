// ad2_tma.cuh — the fused B-ADMM iteration kernel with per-warp TMA (cp.async.bulk) staging.
// Modified B-ADMM of AD2-clustering (arXiv 1510.00012, Alg. 4; "P:n" = PAPER.md line).
//
// Each warp owns a 2-stage shared-memory pipeline.  A pass = G = 32/MP consecutive members of
// one cluster; their Pi / Lambda blocks (contiguous, column-major, leading dimension ld) and
// their support points Y (row stride dy) are brought in by three 1-D bulk copies completing on
// an mbarrier, the next pass's copies are in flight while this pass computes, and the results
// leave by bulk stores from the same shared-memory slots.  The cost C = ||x_i - y_j||^2 is
// recomputed from the staged supports (difference form, d <= DP FMAs per entry) instead of
// being read from HBM, so an iteration moves 16 B per plan entry plus ~dy*4/m B of supports.
#pragma once
#include "ad2_kernels.cuh"

namespace ad2k {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni W%=;\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <typename T, int MP, int NCH, int DP>
struct TmaLayout {
  static constexpr int G = 32 / MP;
  static constexpr int MK = MP * NCH;
  static constexpr int CAP = 32 * MK;          // plan entries staged per pass (G*MP rows x MK cols)
  static constexpr int DYMAX = DP + 16 / (int)sizeof(T);   // Y row: DP coordinates + |y|^2 (+pad)
  static constexpr int YCAP = G * MK * DYMAX;  // support coordinates staged per pass
  static constexpr int STAGE = 2 * CAP + YCAP; // elements: [P|L|Y]
  static constexpr int TILE = MP * 32;
  static constexpr int FB = G * MK;
  static constexpr size_t WARP_BYTES =
      ((sizeof(T) * (size_t)(2 * STAGE + TILE + FB) + 16 + 127) / 128) * 128;
  static constexpr size_t CTA_BYTES = NWARP * WARP_BYTES;
  // static shared memory of the kernel (item-partial combination), for the capacity check
  static constexpr size_t STATIC_BYTES = sizeof(T) * (size_t)NWARP * G * MP * (DP + 1);
};

template <typename T, int MP, int NCH, int MODE, int DP>
__global__ void __launch_bounds__(NWARP * 32)
k_badmm_tma(const IterArgs<T> a) {
  using N = Num<T>;
  using V = typename Vec16<T>::type;
  using Lay = TmaLayout<T, MP, NCH, DP>;
  constexpr int G = Lay::G, MK = Lay::MK, CAP = Lay::CAP;
  constexpr int E = 16 / (int)sizeof(T);
  constexpr int NB = MK / 4;                          // column blocks (warp-uniform skip past m_k)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* wb = reinterpret_cast<T*>(smem_raw + (size_t)warp * Lay::WARP_BYTES);
  T* const sPL = wb;                                   // two stages of [P | L | Y]
  T* const tile = wb + 2 * Lay::STAGE;                 // column-sum transpose tile [MP][32]
  T* const fbuf = tile + Lay::TILE;                    // per-column factors [G][MK]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(
      reinterpret_cast<unsigned char*>(fbuf + Lay::FB) + ((16 - ((uintptr_t)(fbuf + Lay::FB) & 15)) & 15));

  // lane (seg, i): row i of the seg-th member of a pass.  Blocks have ld == MP rows; rows
  // i >= m are zero padding and stay zero (eps_r = 0 there), so no per-entry row predicates.
  const int seg = lane / MP, i = lane - seg * MP;
  const int item = blockIdx.x;
  const int c = a.item_cl[item];
  const int64_t mb = a.item_mb[item], me = a.item_mb[item + 1];
  const int m = a.m, d = a.d, dy = a.dy;
  const bool rowok = i < m;
  const T kx = a.kx[c];
  const T rho = a.rho[c];
  const T eps_r = rowok ? a.eps : T(0);
  const T wi = (MODE != P1ONLY && rowok) ? a.w[(int64_t)c * m + i] : T(0);
  // cost operands: C_ij = (|x_i|^2 + |y_j|^2) + sum_t (-2 x_it) y_jt, |y_j|^2 staged at Y[j][d]
  T xn[DP];
  T xx = T(0);
#pragma unroll
  for (int t = 0; t < DP; ++t) {
    const T v = (rowok && t < d) ? a.x[((int64_t)c * m + i) * d + t] : T(0);
    xx += v * v;
    xn[t] = T(-2) * v;
  }
  T accw = T(0), accm = T(0);
  T accx[(MODE == P2ONLY) ? DP : 1];
#pragma unroll
  for (int t = 0; t < ((MODE == P2ONLY) ? DP : 1); ++t) accx[t] = T(0);
  bool bad = false;

  const T* src_plan = (MODE == P1ONLY) ? a.Q : a.P;
  T* dst_plan = (MODE == P2ONLY) ? a.Q : a.P;
  const int64_t step = (int64_t)NWARP * G;

  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int t) {                            // lane 0 only
    const int64_t k0 = mb + (int64_t)warp * G + (int64_t)t * step;
    if (k0 >= me) return;
    const int64_t k1 = (k0 + G < me) ? k0 + G : me;
    const int64_t p0 = a.off[k0], p1 = a.off[k1];
    const uint32_t bp = (uint32_t)((int64_t)MP * (p1 - p0) * (int64_t)sizeof(T));
    const uint32_t by = (uint32_t)((int64_t)dy * (p1 - p0) * (int64_t)sizeof(T));
    T* st = sPL + (t & 1) * Lay::STAGE;
    mbar_expect_tx(&bar[t & 1], 2 * bp + by);
    tma_load(st, src_plan + (int64_t)MP * p0, bp, &bar[t & 1]);
    tma_load(st + CAP, a.L + (int64_t)MP * p0, bp, &bar[t & 1]);
    tma_load(st + 2 * CAP, a.Y + (int64_t)dy * p0, by, &bar[t & 1]);
  };
  if (lane == 0) issue(0);

  for (int t = 0;; ++t) {
    const int64_t k0 = mb + (int64_t)warp * G + (int64_t)t * step;   // warp-uniform
    if (k0 >= me) break;
    if (lane == 0) {
      bulk_wait_read_all();          // stores of pass t-1 have left the stage about to be refilled
      issue(t + 1);
    }
    const int64_t k1 = (k0 + G < me) ? k0 + G : me;
    const int64_t pbase = a.off[k0];
    const int64_t k = k0 + seg;
    const bool has = k < k1;
    const int64_t o0 = has ? a.off[k] : pbase;
    const int mk = has ? (int)(a.off[k + 1] - o0) : 0;
    const int mkw = (G == 1) ? mk : (int)__reduce_max_sync(0xffffffffu, (unsigned)mk);
    T omv[NCH];                                        // w^(k)_j for the column this lane sums
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) omv[ch] = (ch * MP + i < mk) ? __ldg(a.om + o0 + ch * MP + i) : T(0);
    mbar_wait(&bar[t & 1], (uint32_t)((t >> 1) & 1));
    T* const st = sPL + (t & 1) * Lay::STAGE;
    const int rel = (int)(o0 - pbase);
    T* const Ps = st + MP * rel;
    T* const Ls = st + CAP + MP * rel;
    const T* const Ys = st + 2 * CAP + dy * rel;

    T p[MK], l[MK], q[MK];
#pragma unroll
    for (int jb = 0; jb < NB; ++jb) {
      if (4 * jb >= mkw) break;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = 4 * jb + u;
        p[j] = Ps[j * MP + i];
        l[j] = Ls[j * MP + i];
      }
    }
    if constexpr (MODE == P1ONLY) {
#pragma unroll
      for (int j = 0; j < MK; ++j) q[j] = p[j];                       // Pi2^(0)
    } else {
      // phase 2 of the previous iteration: Eq.badmmc1b (Lambda^n), Eq.badmmc1, Eq.badmm2
      T r = T(0);
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * jb + u;
          const T b = p[j] * N::ex(l[j] * kx) + eps_r;
          q[j] = (j < mk) ? b : T(0);
          r += q[j];
        }
      }
      const T f = (has && rowok) ? wi / r : T(0);
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * jb + u;
          q[j] = q[j] * f;
          l[j] = l[j] + rho * (p[j] - q[j]);
        }
      }
    }
    if constexpr (MODE == P2ONLY) {
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * jb + u;
          if (j < mk) {
            Ps[j * MP + i] = q[j];
            Ls[j * MP + i] = l[j];
            // support-update partials (Eq.updatex, X5): sum_j pi2_ij y_j and sum_j pi2_ij
            accm += q[j];
#pragma unroll
            for (int tt = 0; tt < DP / E; ++tt) {
              const V v = *reinterpret_cast<const V*>(Ys + j * dy + tt * E);
              const T* ve = reinterpret_cast<const T*>(&v);
#pragma unroll
              for (int u2 = 0; u2 < E; ++u2) accx[tt * E + u2] += q[j] * ve[u2];
            }
          }
        }
      }
    } else {
      // phase 1: C_ij, pt2 = Pi2 exp(-(C + Lambda)/rho) + eps (Eq.badmmc0b)
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * jb + u;
          const T* yj = Ys + j * dy;
          T cst = xx + yj[d];
#pragma unroll
          for (int tt = 0; tt < DP / E; ++tt) {
            const V v = *reinterpret_cast<const V*>(yj + tt * E);
            const T* ve = reinterpret_cast<const T*>(&v);
#pragma unroll
            for (int u2 = 0; u2 < E; ++u2) cst = fma(xn[tt * E + u2], ve[u2], cst);
          }
          const T av = q[j] * N::ex(-(cst + l[j]) * kx) + eps_r;
          p[j] = (j < mk) ? av : T(0);
        }
      }
      // column sums (Eq.badmmc0 denominators) through the swizzled transpose tile
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        __syncwarp();
#pragma unroll
        for (int u = 0; u < MP; ++u) {
          if (ch * MP + (u & ~3) >= mkw) break;
          tile[u * 32 + ((((lane / E) ^ (u & 7))) * E) + (lane % E)] = p[ch * MP + u];
        }
        __syncwarp();
        T s = T(0);
#pragma unroll
        for (int cc = 0; cc < MP / E; ++cc) {
          const V v = *reinterpret_cast<const V*>(&tile[i * 32 + ((seg * (MP / E) + cc) ^ (i & 7)) * E]);
          s += Vec16<T>::hsum(v);
        }
        const int jc = ch * MP + i;
        fbuf[seg * MK + jc] = (jc < mk) ? omv[ch] / s : T(0);          // Eq.badmmc0
      }
      __syncwarp();
      T r2 = T(0);
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
        T fe[4];
#pragma unroll
        for (int u = 0; u < 4; u += E) {
          const V fv = *reinterpret_cast<const V*>(&fbuf[seg * MK + 4 * jb + u]);
#pragma unroll
          for (int u2 = 0; u2 < E; ++u2) fe[u + u2] = reinterpret_cast<const T*>(&fv)[u2];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * jb + u;
          p[j] = p[j] * fe[u];
          const T b = p[j] * N::ex(l[j] * kx) + eps_r;                  // Eq.badmmc1b row mass
          r2 += (j < mk) ? b : T(0);
        }
      }
      T R = r2;
#pragma unroll
      for (int h = MP / 2; h >= 1; h >>= 1) R += __shfl_xor_sync(0xffffffffu, R, h);
      if (has && rowok) {
        const T wt = r2 / R;
        accw += (a.rule == 1) ? sqrt(wt) : wt;
        bad |= !isfinite(wt);
      }
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = 4 * jb + u;
          if (j < mk) {
            Ps[j * MP + i] = p[j];
            if (MODE == FUSED) Ls[j * MP + i] = l[j];
          }
        }
      }
    }
    // results leave by bulk stores from the same slots
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      const int64_t p1 = a.off[k1];
      const uint32_t bp = (uint32_t)((int64_t)MP * (p1 - pbase) * (int64_t)sizeof(T));
      tma_store(dst_plan + (int64_t)MP * pbase, st, bp);
      if (MODE != P1ONLY) tma_store(a.L + (int64_t)MP * pbase, st + CAP, bp);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
  if (bad) atomicOr(a.err, ERR_NONFINITE);

  // fixed-order combination of the per-row accumulators -> this item's partial sums
  if constexpr (MODE != P2ONLY) {
    __shared__ T sw[NWARP * G][MP];
    sw[warp * G + seg][i] = accw;
    __syncthreads();
    if (threadIdx.x < m) {
      T s = T(0);
#pragma unroll
      for (int u = 0; u < NWARP * G; ++u) s += sw[u][threadIdx.x];
      a.pw[(int64_t)item * m + threadIdx.x] = s;
    }
  } else {
    __shared__ T sx[NWARP * G][MP][DP + 1];
#pragma unroll
    for (int t = 0; t < DP; ++t) sx[warp * G + seg][i][t] = accx[t];
    sx[warp * G + seg][i][DP] = accm;
    __syncthreads();
    for (int v = threadIdx.x; v < m * (d + 1); v += NWARP * 32) {
      const int ii = v / (d + 1), t = v - ii * (d + 1);
      const int tt = (t == d) ? DP : t;
      T s = T(0);
#pragma unroll
      for (int u = 0; u < NWARP * G; ++u) s += sx[u][ii][tt];
      a.px[(int64_t)item * m * (d + 1) + v] = s;
    }
  }
}

}  // namespace ad2k
