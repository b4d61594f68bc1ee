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

// ---- tcgen05 pieces of the tensor-core cost (TC instantiation, see k_badmm_tma) ----
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// shared-memory matrix descriptor, K-major without swizzle: 8-row core matrices of 16-byte rows,
// LBO = byte stride between the two K-adjacent core matrices of an MMA, SBO = between 8-row groups
__device__ __forceinline__ uint64_t tc_desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// instruction descriptor kind::tf32: D fp32, A/B tf32, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t tc_idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
// D[tmem] (+)= A[tmem] . B[smem]^T, issued by one thread
__device__ __forceinline__ void tc_mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}
// tf32 split: hi keeps the 10 stored mantissa bits (the MMA reads tf32 by truncation), lo = v - hi
__device__ __forceinline__ float tc_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

template <typename T, int MP, int NCH, int DP>
struct TmaLayout {
  static constexpr int G = 32 / MP;
  static constexpr int MK = MP * NCH;
  static constexpr int E = 16 / (int)sizeof(T);
  // Y row = [y_0..y_{d-1}, 0.., |y|^2 at YYI, 0..] with DY elements (16-byte multiple)
  static constexpr int DY = (DP == 4) ? 4 : DP + E;
  static constexpr int YYI = (DP == 4) ? 3 : DP;
  // one pass = [P block | L block | Y block] of G consecutive members, placed in a per-warp ring
  static constexpr int MAXPASS = (2 * MP + DY) * G * MK;            // elements
  // regions alternate between the ring's start and its end, so the next pass can be placed while
  // the current one computes unless both are unusually large (~2% of passes at m_k ~ Poisson(20))
  static constexpr int RING = ((5 * MAXPASS / 3) + 63) / 64 * 64;
  // in-bounds over-reads past a pass region: G == 1 reads at most 3 masked columns past m_k
  static constexpr int SLACK = ((G == 1 ? 4 * DY : MK * DY + MP * MK) + 63) / 64 * 64;
  static constexpr int TILE = (G == 1) ? 0 : MP * 32;               // G == 1: tile = the pass's P slot
  static constexpr int FB = 2 * G * MK;                            // column factors + log-factors
  // + three mbarriers (the 2-stage load pipeline and, for the tensor-core cost, the MMA)
  static constexpr size_t WARP_BYTES =
      ((sizeof(T) * (size_t)(RING + SLACK + TILE + FB) + 24 + 127) / 128) * 128;
  static constexpr size_t CTA_BYTES = NWARP * WARP_BYTES;
  // static shared memory of the kernel (item-partial combination), for the capacity check
  static constexpr size_t STATIC_BYTES = sizeof(T) * (size_t)NWARP * G * MP * (DP + 1);
};

// pair arithmetic: packed f32x2 (FADD2/FMUL2/FFMA2, sm_100) for fp32, componentwise for fp64
template <typename T> struct Pr;
template <> struct Pr<float> {
  using t = float2;
  static __device__ __forceinline__ float2 make(float a, float b) { return make_float2(a, b); }
  static __device__ __forceinline__ float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
  static __device__ __forceinline__ float2 mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
  static __device__ __forceinline__ float2 fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
};
template <> struct Pr<double> {
  using t = double2;
  static __device__ __forceinline__ double2 make(double a, double b) { return make_double2(a, b); }
  static __device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ double2 mul(double2 a, double2 b) { return make_double2(a.x * b.x, a.y * b.y); }
  static __device__ __forceinline__ double2 fma(double2 a, double2 b, double2 c) {
    return make_double2(::fma(a.x, b.x, c.x), ::fma(a.y, b.y, c.y));
  }
};

// TCC = 1 (fp32, 32-row single-member passes, 4 < d <= 16): the cost's dot products run on the
// tensor cores.  Per CTA, the centroid rows centred on their mean, x'_i = x_i - o, scaled by -2 and
// split into tf32 hi / lo, sit in TMEM (every warp writes them into its own 32 lanes, so rows
// 32 w + i of the M = 128 operand are x'_i for warp w); per member pass, the warp writes its
// points y'_j = y_j - o (hi / lo, canonical K-major layout) into the pass's P and L slots, which
// are free once the state is in registers, and one lane issues 6 tcgen05.mma kind::tf32 (hi.hi,
// hi.lo, lo.hi over K = 16) into the warp's 32 TMEM columns; sweep 2 reads
// D_ij = -2 x'_i . y'_j with tcgen05.ld and forms C_ij = |x'_i|^2 + |y'_j|^2 + D_ij (C is
// translation invariant; centring keeps the products at the scale of C).
// resident CTAs per SM the kernel is compiled for (register cap 65536 / (128 x this)): 4 for the
// fp32 16-row single-chunk small-d passes (118-124 registers, no spill; a small batch such as
// config 2 is latency-bound at 3 warps per scheduler), else 3 (the others would spill at 128)
template <typename T, int MP, int NCH, int DP>
constexpr int tma_min_blocks() {
  return (sizeof(T) == 4 && MP == 16 && NCH == 1 && DP == 4) ? AD2_TMA_MINB16 : 3;
}

template <typename T, int MP, int NCH, int MODE, int DP, int TCC = 0>
__global__ void __launch_bounds__(NWARP * 32, (tma_min_blocks<T, MP, NCH, DP>()))
k_badmm_tma(const IterArgs<T> a) {
  using N = Num<T>;
  using V = typename Vec16<T>::type;
  using PR = Pr<T>;
  using T2 = typename PR::t;
  using Lay = TmaLayout<T, MP, NCH, DP>;
  constexpr int G = Lay::G, MK = Lay::MK, DY = Lay::DY, YYI = Lay::YYI, RING = Lay::RING;
  constexpr int E = Lay::E;
  constexpr int NB = MK / 4;                          // column blocks of 4 (2 pairs), skipped past m_k
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* wb = reinterpret_cast<T*>(smem_raw + (size_t)warp * Lay::WARP_BYTES);
  T* const ring = wb;                                  // per-warp ring of pass regions [P|L|Y]
  T* const tile_sep = wb + RING + Lay::SLACK;          // G > 1: column-sum transpose tile [MP][32]
  T* const fbuf = tile_sep + Lay::TILE;                // per-column factors [G][MK]
  T* const cbuf = fbuf + G * MK;                       // compressed state: column log-factors [G][MK]
  uint64_t* const bar = reinterpret_cast<uint64_t*>(
      reinterpret_cast<unsigned char*>(fbuf + Lay::FB) + ((16 - ((uintptr_t)(fbuf + Lay::FB) & 15)) & 15));

  // Lane (seg, i) = row i of the seg-th member of a pass.  Blocks have MP rows; rows i >= m are
  // zero padding that stays zero (eps_r = 0 there).  Columns j >= m_k of a block are masked at
  // load (p = Lambda = 0) and contribute exactly 0 to every sum: row masses are formed as
  // sum_j p_j e_j + m_k eps (= sum over the m_k real columns of (p_j e_j + eps)).
  const int seg = lane / MP, i = lane - seg * MP;
  const int item = a.perm ? a.perm[blockIdx.x] : (int)blockIdx.x;
  const int c = a.item_cl[item];
  const int64_t mb = a.item_mb[item], me = a.item_mb[item + 1];
  const int m = a.m, d = a.d;
  const bool rowok = i < m;
  const T kx = a.kx[c];
  const T rho = a.rho[c];
  const T eps_r = rowok ? a.eps : T(0);
  constexpr bool PH1 = (MODE == P1ONLY || MODE == P1INIT);   // phase 1 only
  constexpr bool INIT = (MODE == P1INIT);
  // launched as a programmatic dependent of the consensus kernel: everything above (geometry, x,
  // rho) is fixed within a step; w and the plan state are the predecessors' results
  pdl_wait();
  const T wi = (MODE != P1ONLY && rowok) ? a.w[(int64_t)c * m + i] : T(0);
  // Lambda is stored pre-scaled, L' = Lambda * kx (kx = log2(e)/rho for fp32, 1/rho for fp64), so
  // exp(Lambda/rho) = ex(L') and Eq.badmm2 becomes L' += kappa (Pi1 - Pi2) with kappa = kx * rho
  // (log2(e) or 1); ad2_get_plans divides by kx on read-back
  (void)rho;
  const T kap = N::kappa();
  const T2 nkx2 = PR::make(-kx, -kx), rho2 = PR::make(kap, kap);
  const T2 nrho2 = PR::make(-kap, -kap), eps2 = PR::make(eps_r, eps_r);
  // cost C_ij = (|x_i|^2 + |y_j|^2) + sum_t (-2 x_it) y_jt, coordinates taken in pairs
  T2 xn2[DP / 2];
  T xx = T(0);
#pragma unroll
  for (int t = 0; t < DP / 2; ++t) {
    const T v0 = (rowok && 2 * t < d) ? a.x[((int64_t)c * m + i) * d + 2 * t] : T(0);
    const T v1 = (rowok && 2 * t + 1 < d) ? a.x[((int64_t)c * m + i) * d + 2 * t + 1] : T(0);
    xx += v0 * v0;
    xx += v1 * v1;
    xn2[t] = PR::make(T(-2) * v0, T(-2) * v1);
  }
  T accw = T(0), accm = T(0);
  constexpr bool PH2 = (MODE == P2ONLY || MODE == P2X);     // phase 2 only (+ x partials)
  constexpr bool TC = TCC != 0 && sizeof(T) == 4 && MP == 32 && NCH == 1 && DP == 16 && !PH2;
  T* const yyb = fbuf;                                       // TC: |y'_j|^2 of the pass (fbuf is free in sweep 2)
  __shared__ uint32_t tm_s[2];                               // TC: TMEM bases of D (128 columns) and A (32)
  uint32_t tm_d = 0, tm_a = 0;
  float4 oq = make_float4(0.f, 0.f, 0.f, 0.f);               // TC: centre coordinates 4q .. 4q+3 (q = lane & 3)
  if constexpr (TC) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tm_s[0])));
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tm_s[1])));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // centre o = mean of the m centroid rows; A row i = -2 (x_i - o), tf32 hi in columns 0..15 and
    // lo in 16..31; |x_i - o|^2 in fp32 replaces |x_i|^2
    float xv[16], o[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      xv[t] = (rowok && t < d) ? (float)a.x[((int64_t)c * m + i) * d + t] : 0.f;
      float s = xv[t];
#pragma unroll
      for (int h = 16; h >= 1; h >>= 1) s += __shfl_xor_sync(0xffffffffu, s, h);
      o[t] = s / (float)m;
    }
    uint32_t r[32];
    float xc = 0.f;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const float v = (rowok && t < d) ? xv[t] - o[t] : 0.f;
      xc = fmaf(v, v, xc);
      const float av = -2.f * v, h = tc_hi(av);
      r[t] = __float_as_uint(h);
      r[16 + t] = __float_as_uint(av - h);
    }
    xx = (T)xc;
    const int q = lane & 3;
    oq.x = q == 0 ? o[0] : q == 1 ? o[4] : q == 2 ? o[8] : o[12];
    oq.y = q == 0 ? o[1] : q == 1 ? o[5] : q == 2 ? o[9] : o[13];
    oq.z = q == 0 ? o[2] : q == 1 ? o[6] : q == 2 ? o[10] : o[14];
    oq.w = q == 0 ? o[3] : q == 1 ? o[7] : q == 2 ? o[11] : o[15];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    tm_d = tm_s[0];
    tm_a = tm_s[1];
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tm_a + ((uint32_t)(32 * warp) << 16)),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();                                         // all 128 A lanes written before any MMA reads them
    tc_fence_after();
  }
  uint32_t mph = 0;                                          // TC: phase of the MMA mbarrier
  constexpr bool XP = (MODE == FUSEDX || MODE == GXOUT);     // FUSED + x partials
  constexpr bool GI = (MODE == GIN);                          // compressed state: anchor launch
  constexpr bool GC = (MODE == GMID || MODE == GXOUT);       // phase 2 from (G, U, ra, cb)
  constexpr bool GW = (MODE == GIN || MODE == GMID);         // phase 1 stores (U, ra, cb)
  constexpr int FM = (XP || GI || GC) ? FUSED : MODE;        // the mode the sweeps follow
  // FUSEDX recomputes pe = Pi1 exp(Lambda/rho) in the second sweep instead of keeping it from the
  // first (one more exp per entry, 32 fewer registers: 3 CTAs per SM instead of 2, same values)
  constexpr bool RECOMP = (MODE == FUSEDX);
  constexpr bool NOSTORE = (MODE == P2X);
  T accx[(PH2 || XP) ? DP : 1];
  T2 accy[XP ? DP / 2 : 1];                                  // FUSEDX: the member's sum (pe + eps) y
#pragma unroll
  for (int t = 0; t < ((PH2 || XP) ? DP : 1); ++t) accx[t] = T(0);
#pragma unroll
  for (int t = 0; t < (XP ? DP / 2 : 1); ++t) accy[t] = PR::make(T(0), T(0));
  bool bad = false;

  const T* src_plan = (MODE == P1ONLY || GC) ? a.Q : a.P;     // GC: the anchor G lives in Q
  T* dst_plan = (MODE == P2ONLY || GI) ? a.Q : a.P;
  const T gsn = -(T)a.gs;                                       // GC: -(iterations since the anchor)
  bool epshit = false;
  const int64_t step = (int64_t)NWARP * G;

  // ring (and its over-read slack) zeroed once: every value it ever holds is then finite
  for (int e = lane * E; e < RING + Lay::SLACK; e += 32 * E) *reinterpret_cast<V*>(ring + e) = V{};
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    if constexpr (TC) mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  __syncwarp();
  // pass geometry (warp-uniform): points [p0, p1) of members [k0, k1)
  auto pass_pts = [&](int t, int64_t& p0, int64_t& p1) -> int {
    const int64_t k0 = mb + (int64_t)warp * G + (int64_t)t * step;
    if (k0 >= me) return 0;
    const int64_t k1 = (k0 + G < me) ? k0 + G : me;
    p0 = a.off[k0];
    p1 = a.off[k1];
    return (int)(p1 - p0);
  };
  // G == 1: the slots of a pass region hold ceil4(m_k) columns ([P | L | Y] at 0, MP*np4,
  // 2*MP*np4); the 0-3 padding columns of P and L are zeroed by the lanes, so the column blocks
  // of 4 need no masks and the stores no predicates.  G > 1: packed slots, masked blocks.
  constexpr bool PAD = (G == 1);
  auto slot = [](int np) { return PAD ? ((np + 3) & ~3) : np; };
  auto issue = [&](int t, int base, int64_t p0, int np) {              // lane 0 only
    const uint32_t bp = (uint32_t)(MP * np * (int)sizeof(T));
    const uint32_t by = (uint32_t)(DY * np * (int)sizeof(T));
    const int ns = slot(np);
    T* st = ring + base;
    mbar_expect_tx(&bar[t & 1], INIT ? by : 2 * bp + by);
    if constexpr (INIT) {
      tma_load(st + 2 * MP * ns, a.Y + (int64_t)DY * p0, by, &bar[t & 1]);
    } else {
      tma_load(st, src_plan + (int64_t)MP * p0, bp, &bar[t & 1]);
      tma_load(st + MP * ns, a.L + (int64_t)MP * p0, bp, &bar[t & 1]);
      tma_load(st + 2 * MP * ns, a.Y + (int64_t)DY * p0, by, &bar[t & 1]);
    }
  };
  int64_t cp0 = 0, cp1 = 0;
  int cnp = pass_pts(0, cp0, cp1);
  // the geometry of pass t+1 is loaded one pass ahead (its offsets are on the critical path of
  // the ring placement): pass t uses (np0, nnp) loaded during pass t-1
  int64_t np0 = 0, np1 = 0;
  int nnp = pass_pts(1, np0, np1);
  int cbase = 0;                                       // ring offset of the current pass
  if (lane == 0 && cnp > 0) issue(0, 0, cp0, cnp);
  // GC: the member's log-factors (global loads) are fetched one pass ahead for G == 1, so their
  // latency hides behind a pass instead of stalling the start of the next one
  const T lgw = (GC && rowok && wi > T(0)) ? N::lg(wi) : T(0);
  T pf_cb[NCH], pf_ra = T(0), pf_om[NCH];
  if constexpr (G == 1) {                              // w^(k)_j of the first pass (then one ahead)
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) pf_om[ch] = (ch * MP + i < cnp) ? __ldg(a.om + cp0 + ch * MP + i) : T(0);
  }
  if constexpr (GC && G == 1) {
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) pf_cb[ch] = (ch * MP + i < cnp) ? a.cb[cp0 + ch * MP + i] : T(0);
    if (cnp > 0 && rowok) pf_ra = a.ra[(mb + warp) * MP + i];
  }

  for (int t = 0; cnp > 0; ++t) {
    // place pass t+1 behind pass t (or at the ring start) while t computes
    int64_t fp0 = 0, fp1 = 0;
    const int fnp = pass_pts(t + 2, fp0, fp1);          // consumed next pass
    const int csize = (2 * MP + DY) * slot(cnp), nsize = (2 * MP + DY) * slot(nnp);
    int nbase = -1;
    if (nnp > 0) {
      if (cbase == 0) {                                // current at the start: next end-aligned
        if (RING - nsize >= csize) nbase = RING - nsize;
      } else if (nsize <= cbase) {                     // current end-aligned: next at the start
        nbase = 0;
      }
    }
    // the current and the next pass regions lie inside the ring and do not overlap; a pass never
    // holds more than G members of at most MK columns
    AD2_CHECK(cnp <= G * MK && nnp <= G * MK && cbase >= 0 && cbase + csize <= RING);
    AD2_CHECK(nbase < 0 || (nbase + nsize <= RING && (nbase >= cbase + csize || nbase + nsize <= cbase)));
    if (lane == 0 && nbase >= 0) {
      bulk_wait_read_all();          // pass t-1 has left its region
      issue(t + 1, nbase, np0, nnp);
    }
    const int64_t k0 = mb + (int64_t)warp * G + (int64_t)t * step;
    const int64_t k1 = (k0 + G < me) ? k0 + G : me;
    const int64_t k = k0 + seg;
    const bool has = k < k1;
    int64_t o0 = cp0;
    int mk = cnp;                                      // G == 1: the member is the pass
    if constexpr (G > 1) {
      o0 = has ? a.off[k] : cp0;
      mk = has ? (int)(a.off[k + 1] - o0) : 0;
    }
    const int mkw = (G == 1) ? mk : (int)__reduce_max_sync(0xffffffffu, (unsigned)mk);
    AD2_CHECK(mk >= 0 && mk <= MK && mkw <= MK);
    const T mkeps = (T)mk * eps_r;
    T omv[NCH];                                        // w^(k)_j for the column this lane sums
    if constexpr (G == 1) {                            // prefetched one pass ahead
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        omv[ch] = pf_om[ch];
        pf_om[ch] = (ch * MP + i < nnp) ? __ldg(a.om + np0 + ch * MP + i) : T(0);
      }
    } else {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) omv[ch] = (ch * MP + i < mk) ? __ldg(a.om + o0 + ch * MP + i) : T(0);
    }
    T cbv[NCH];                                        // compressed state: this lane's column log-factor
    T rowexp = T(0);                                   // GC: log-factor of row i, incl. w^{t-1}_i
    if constexpr (GC) {
      T rav = T(0);
      if constexpr (G == 1) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) cbv[ch] = pf_cb[ch];
        rav = pf_ra;
        const int64_t kn = k + step;                   // the next pass's member
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) pf_cb[ch] = (ch * MP + i < nnp) ? a.cb[np0 + ch * MP + i] : T(0);
        pf_ra = (nnp > 0 && rowok) ? a.ra[kn * MP + i] : T(0);
      } else {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) cbv[ch] = (ch * MP + i < mk) ? a.cb[o0 + ch * MP + i] : T(0);
        if (has && rowok) rav = a.ra[k * MP + i];
      }
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) cbuf[seg * MK + ch * MP + i] = cbv[ch];
      if (has && rowok) rowexp = rav + lgw;
      __syncwarp();                                    // cbuf complete before the sweeps read it
    } else {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) cbv[ch] = T(0);
    }
    mbar_wait(&bar[t & 1], (uint32_t)((t >> 1) & 1));
    T* const st = ring + cbase;
    const int rel = (int)(o0 - cp0);
    const int cns = slot(cnp);
    T* const Ps = st + MP * rel;
    T* const Ls = st + MP * cns + MP * rel;
    const T* const Ys = st + 2 * MP * cns + DY * rel;
    if constexpr (PAD && !INIT) {
      // G == 1 blocks use the pair layout (blk_idx, ad2_kernels.cuh): columns 2q, 2q+1 interleaved
      // by row, so a lane moves both with one 8-byte access; an odd m_k's last column arrives in the
      // single-column layout and is rewritten here as the pair (m_k - 1, pad) with a zero partner
      // (a lane only ever touches its own row's pairs below and in sweep 1: one __syncwarp, between
      // the single-layout reads of the odd column and the pair writes over them)
      const bool odd = mk & 1;
      const int mk2 = (mk + 1) & ~1;                   // columns [mk2, cns): one padding pair, or none
      T* const po = Ps + (mk - 1) * MP;
      T* const lo = Ls + (mk - 1) * MP;
      T px = T(0), lx = T(0);
      if (odd) {
        px = po[i];
        lx = lo[i];
      }
      if (mk2 < cns) {                                 // p = Lambda = 0
        *reinterpret_cast<T2*>(Ps + mk2 * MP + 2 * i) = PR::make(T(0), T(0));
        *reinterpret_cast<T2*>(Ls + mk2 * MP + 2 * i) = PR::make(T(0), T(0));
      }
      __syncwarp();
      if (odd) {
        *reinterpret_cast<T2*>(po + 2 * i) = PR::make(px, T(0));
        *reinterpret_cast<T2*>(lo + 2 * i) = PR::make(lx, T(0));
      }
    }
    T* const tile = (G == 1) ? st : tile_sep;          // G == 1: reuse this pass's P slot
    // fp32 single-member passes: the tile has rows of 36 (column jt at jt*36: conflict-free 4-byte
    // stores, lane i reads its column with 16-byte loads at i*36 + 4cc, banks 4i .. 4i+3 per
    // quarter warp); 36 m_k <= 64 ns floats, so it stays inside the P and L slots, both free
    // between sweep 2 and sweep 3 (the state is in registers)
    constexpr bool TPAD = PAD && (E == 4) && MP == 32;

    T2 p2[MK / 2], l2[MK / 2], q2[MK / 2];
    // ---- load (columns >= m_k masked to 0) and, unless P1ONLY, the first half of phase 2:
    //      pe = Pi1 exp(Lambda/rho) (Eq.badmmc1b without eps), r = sum_j pe_j + m_k eps
    T2 racc[2] = {PR::make(T(0), T(0)), PR::make(T(0), T(0))};
    auto ph2_first = [&](int jp, int h) {
      if constexpr (PH1 || GC) {
        q2[jp] = p2[jp];                                               // Pi2^(0) / unused (GC)
      } else if constexpr (RECOMP) {
        const T2 e = PR::make(N::ex(l2[jp].x), N::ex(l2[jp].y));
        racc[h] = PR::add(racc[h], PR::mul(p2[jp], e));
      } else {
        const T2 e = PR::make(N::ex(l2[jp].x), N::ex(l2[jp].y));
        q2[jp] = PR::mul(p2[jp], e);
        racc[h] = PR::add(racc[h], q2[jp]);
      }
    };
#pragma unroll
    for (int jb = 0; jb < NB; ++jb) {
      if (4 * jb >= mkw) break;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jp = 2 * jb + h, j = 2 * jp;
        if constexpr (INIT) {                          // Pi2^0 = w_i w_j^(k), Lambda = 0
          const T o0v = j < mk ? __ldg(a.om + o0 + j) : T(0);
          const T o1v = j + 1 < mk ? __ldg(a.om + o0 + j + 1) : T(0);
          p2[jp] = PR::make(wi * o0v, wi * o1v);
          l2[jp] = PR::make(T(0), T(0));
        } else if constexpr (PAD) {                    // pair layout: one 8-byte load per pair
          p2[jp] = *reinterpret_cast<const T2*>(Ps + j * MP + 2 * i);
          l2[jp] = *reinterpret_cast<const T2*>(Ls + j * MP + 2 * i);
        } else {
          const bool v0 = j < mk, v1 = j + 1 < mk;
          const T pa = Ps[j * MP + i], pb = Ps[(j + 1) * MP + i];
          const T la = Ls[j * MP + i], lb = Ls[(j + 1) * MP + i];
          p2[jp] = PR::make(v0 ? pa : T(0), v1 ? pb : T(0));
          l2[jp] = PR::make(v0 ? la : T(0), v1 ? lb : T(0));
        }
        if constexpr (!TC) ph2_first(jp, h);
      }
    }
    if constexpr (TC) {
      // the state is in registers: the P and L slots take the B operand, y'_j = y_j - o split into
      // tf32 hi / lo, point j coordinates 4q..4q+3 at byte (j/8)*512 + q*128 + (j%8)*16 (8-row core
      // matrices; rows j >= m_k are zero, so padding columns see C = |x'_i|^2)
      T* const Bh = st;
      const int g8 = (cnp + 7) >> 3;
      T* const Bl = Bh + g8 * 128;
      const int q = lane & 3, jr = lane >> 2;
      __syncwarp();
      for (int r = 0; r < g8; ++r) {
        const int j = 8 * r + jr;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < cnp) {
          v = *reinterpret_cast<const float4*>(Ys + j * DY + 4 * q);
          v.x -= oq.x; v.y -= oq.y; v.z -= oq.z; v.w -= oq.w;
        }
        const float4 hv = make_float4(tc_hi(v.x), tc_hi(v.y), tc_hi(v.z), tc_hi(v.w));
        const float4 lv = make_float4(v.x - hv.x, v.y - hv.y, v.z - hv.z, v.w - hv.w);
        *reinterpret_cast<float4*>(Bh + r * 128 + q * 32 + jr * 4) = hv;
        *reinterpret_cast<float4*>(Bl + r * 128 + q * 32 + jr * 4) = lv;
        float s = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, v.w * v.w)));
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (q == 0) yyb[j] = s;
      }
      fence_proxy_async_smem();                        // generic writes -> tensor core (async proxy)
      tc_fence_before();                               // the previous pass's tcgen05.ld are complete
      __syncwarp();
      if (lane == 0) {
        tc_fence_after();
        const uint32_t dcol = tm_d + 32 * warp;
        const uint32_t idesc = cnp <= 16 ? tc_idesc_tf32(16) : tc_idesc_tf32(32);
        const uint64_t dh = tc_desc_kmajor(smem_u32(Bh), 128, 512), dl = tc_desc_kmajor(smem_u32(Bl), 128, 512);
        // K = 16 in two MMAs of 8 (+256 bytes = +16 in the descriptor's address field): hi.hi,
        // hi.lo, lo.hi, issued from one asm block (one set of uniform operands)
        asm volatile(
            "{\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 h1, l1;\n\t.reg .pred p0, p1;\n\t"
            "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
            "add.u64 h1, %2, 16;\n\tadd.u64 l1, %3, 16;\n\t"
            "setp.ne.b32 p0, 0, 0;\n\tsetp.eq.b32 p1, 0, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], h1, %4, p1;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %4, p1;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [a1], l1, %4, p1;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [a2], %2, %4, p1;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [a3], h1, %4, p1;\n\t"
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}" ::"r"(dcol),
            "r"(tm_a), "l"(dh), "l"(dl), "r"(idesc), "r"(smem_u32(&bar[2]))
            : "memory");
      }
      __syncwarp();
      // the first half of phase 2 runs while the tensor core works
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) ph2_first(2 * jb + h, h);
      }
    }
    T f = T(0);
    if constexpr (!PH1 && !GC) {
      const T r = (racc[0].x + racc[1].x) + (racc[0].y + racc[1].y) + mkeps;
      f = (has && rowok) ? N::div(wi, r) : T(0);                    // Eq.badmmc1: w_i / rowsum
    }
    const T2 f2 = PR::make(f, f), ef2 = PR::make(eps_r * f, eps_r * f);

    if constexpr (PH2) {
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int jp = 2 * jb + h, j = 2 * jp;
          const T2 q = PR::fma(q2[jp], f2, ef2);                        // Pi2 = (pe + eps) w_i / r
          const T2 l = PR::fma(nrho2, q, PR::fma(rho2, p2[jp], l2[jp]));  // Eq.badmm2
          if constexpr (PAD && !NOSTORE) {
            *reinterpret_cast<T2*>(Ps + j * MP + 2 * i) = q;
            *reinterpret_cast<T2*>(Ls + j * MP + 2 * i) = l;
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int jj = j + u;
            const T qv = u ? q.y : q.x, lv = u ? l.y : l.x;
            if (!PAD && !NOSTORE && jj < mk) {   // packed blocks (G > 1): no tail writes
              Ps[jj * MP + i] = qv;
              Ls[jj * MP + i] = lv;
            }
            if (jj < mk) {                   // support-update partials (Eq.updatex, X5)
              accm += qv;
#pragma unroll
              for (int tt = 0; tt < DP / E; ++tt) {
                const V v = *reinterpret_cast<const V*>(Ys + jj * DY + tt * E);
                const T* ve = reinterpret_cast<const T*>(&v);
#pragma unroll
                for (int u2 = 0; u2 < E; ++u2) accx[tt * E + u2] += qv * ve[u2];
              }
            }
          }
        }
      }
    } else {
      // ---- rest of phase 2 (FUSED) and phase 1, four columns at a time:
      //      C_ij; pt2 = Pi2 exp(-(C + Lambda)/rho) + eps (Eq.badmmc0b) -> tile
      if constexpr (TC) {                                // the pass's MMAs have landed in TMEM
        mbar_wait(&bar[2], mph);
        mph ^= 1;
        tc_fence_after();
      }
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
        T2 c2[4];
        if constexpr (TC) {
          // (|x'_i|^2 + |y'_j|^2, -2 x'_i . y'_j): row i of the warp's TMEM lanes, columns 4jb..4jb+3
          uint32_t dv[4];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(dv[0]), "=r"(dv[1]), "=r"(dv[2]), "=r"(dv[3])
                       : "r"(tm_d + ((uint32_t)(32 * warp) << 16) + (uint32_t)(32 * warp + 4 * jb)));
          const float4 yv = *reinterpret_cast<const float4*>(&yyb[4 * jb]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          c2[0] = PR::make(xx + (T)yv.x, (T)__uint_as_float(dv[0]));
          c2[1] = PR::make(xx + (T)yv.y, (T)__uint_as_float(dv[1]));
          c2[2] = PR::make(xx + (T)yv.z, (T)__uint_as_float(dv[2]));
          c2[3] = PR::make(xx + (T)yv.w, (T)__uint_as_float(dv[3]));
        } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) c2[u] = PR::make(xx, Ys[(4 * jb + u) * DY + YYI]);   // (|x|^2, |y|^2) + dot pairs
#pragma unroll
        for (int tt = 0; tt < DP / E; ++tt) {
          V v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const V*>(Ys + (4 * jb + u) * DY + tt * E);
#pragma unroll
          for (int u2 = 0; u2 < E / 2; ++u2)
#pragma unroll
            for (int u = 0; u < 4; ++u)
              c2[u] = PR::fma(xn2[tt * (E / 2) + u2], reinterpret_cast<const T2*>(&v[u])[u2], c2[u]);
        }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int jp = 2 * jb + h, j = 2 * jp;
          T2 q = q2[jp];
          const T2 cst = PR::make(c2[2 * h].x + c2[2 * h].y, c2[2 * h + 1].x + c2[2 * h + 1].y);
          if constexpr (GC) {
            // Pi2^{t-1} = G exp(rowexp_i + cb_j - s C kx) (P4), Lambda^{t-1} = U - rho Pi2^{t-1}
            const T2 cbj = *reinterpret_cast<const T2*>(&cbuf[seg * MK + j]);
            const T2 ck = PR::mul(cst, PR::make(kx, kx));
            const T2 ex = PR::fma(ck, PR::make(gsn, gsn), PR::add(PR::make(rowexp, rowexp), cbj));
            q = PR::mul(p2[jp], PR::make(N::ex(ex.x), N::ex(ex.y)));
            l2[jp] = PR::fma(nrho2, q, l2[jp]);
          } else if constexpr (FM == FUSED) {
            if constexpr (RECOMP) q = PR::mul(p2[jp], PR::make(N::ex(l2[jp].x), N::ex(l2[jp].y)));
            q = PR::fma(RECOMP ? q : q2[jp], f2, ef2);                    // Pi2 (Eq.badmmc1)
            l2[jp] = PR::fma(nrho2, q, PR::fma(rho2, p2[jp], l2[jp]));     // Eq.badmm2
            if constexpr (GI) q2[jp] = q;                                  // the anchor G, stored below
          }
          const T2 ar = PR::fma(cst, nkx2, PR::make(-l2[jp].x, -l2[jp].y));   // -(C kx + L')
          const T2 e = PR::make(N::ex(ar.x), N::ex(ar.y));
          p2[jp] = PR::fma(q, e, eps2);                                    // pt2 (column j >= m_k: finite)
        }
      }
      // column sums over the m rows (Eq.badmmc0 denominators) through the swizzled tile
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        __syncwarp();                                                    // P slot / tile free
#pragma unroll
        for (int jb = ch * (MP / 4); jb < (ch + 1) * (MP / 4); ++jb) {
          if (4 * jb >= mkw) break;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = 4 * jb + u, jt = j - ch * MP;
            const T v = (u & 1) ? p2[j / 2].y : p2[j / 2].x;
            if constexpr (TPAD) {
              tile[jt * 36 + lane] = v;                // padded rows: immediate offsets, no conflicts
            } else {
              // swizzle ((lane / E) ^ (jt & 7)) * E + lane % E == lane ^ ((jt & 7) * E) (E a power of 2)
              if (PAD || j < mkw) tile[jt * 32 + (lane ^ ((jt & 7) * E))] = v;   // P slot bound
            }
          }
        }
        __syncwarp();
        const int jc = ch * MP + i;
        T s = T(1);
        if (jc < mk) {                 // packed pairwise tree over the MP row values
          T2 sp[MP / E];
#pragma unroll
          for (int cc = 0; cc < MP / E; ++cc) {
            const V v = TPAD ? *reinterpret_cast<const V*>(&tile[i * 36 + cc * E])
                             : *reinterpret_cast<const V*>(&tile[i * 32 + (((seg * (MP / E) + cc) * E) ^ ((i & 7) * E))]);
            const T2* v2 = reinterpret_cast<const T2*>(&v);
            sp[cc] = (E == 4) ? PR::add(v2[0], v2[(E == 4) ? 1 : 0]) : v2[0];
          }
#pragma unroll
          for (int w = MP / E / 2; w >= 1; w >>= 1)
#pragma unroll
            for (int cc = 0; cc < w; ++cc) sp[cc] = PR::add(sp[cc], sp[cc + w]);
          s = sp[0].x + sp[0].y;
        }
        const T fcol = (jc < mk) ? N::div(omv[ch], s) : T(0);           // Eq.badmmc0: w_j^(k) / colsum
        fbuf[seg * MK + jc] = fcol;
        if constexpr (GW) {
          if (jc < mk) a.cb[o0 + jc] = cbv[ch] + N::lg(fcol);             // b_j *= w_j / colsum_j
        }
        if constexpr (GC) {
          // the column's mass is the eps floor's, so the eps-free recursion is off by up to the
          // column's weight w_j^(k): flagged when that weight is not negligible (>= 1e-7 of the
          // member's mass; Dirichlet weights far below it are common and move nothing)
          if (jc < mk && s <= T(2) * (T)m * a.eps && omv[ch] >= T(1e-7)) epshit = true;
        }
      }
      __syncwarp();
      // ---- Pi1 = pt2 * factor_j; pt1 = Pi1 exp(Lambda/rho) + eps (Eq.badmmc1b) row masses
      T2 racc2[2] = {PR::make(T(0), T(0)), PR::make(T(0), T(0))};
#pragma unroll
      for (int jb = 0; jb < NB; ++jb) {
        if (4 * jb >= mkw) break;
        const V fv = *reinterpret_cast<const V*>(&fbuf[seg * MK + 4 * jb]);
        const T2* fp = reinterpret_cast<const T2*>(&fv);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int jp = 2 * jb + h, j = 2 * jp;
          const T2 fj = (E == 4) ? fp[h] : *reinterpret_cast<const T2*>(&fbuf[seg * MK + j]);
          p2[jp] = PR::mul(p2[jp], fj);
          const T2 e = PR::make(N::ex(l2[jp].x), N::ex(l2[jp].y));
          if constexpr (XP) {
            // x partials of the coming Pi2 (see below): sum_j (pe_ij + eps) y_j, scaled by 1/r_i later
            const T2 pe = PR::mul(p2[jp], e);
            racc2[h] = PR::add(racc2[h], pe);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int jj = j + u;
              const T qv = (jj < mk) ? (u ? pe.y : pe.x) + eps_r : T(0);   // masked column: adds exactly 0
              const T2 qv2 = PR::make(qv, qv);
#pragma unroll
              for (int tt = 0; tt < DP / E; ++tt) {
                const V v = *reinterpret_cast<const V*>(Ys + jj * DY + tt * E);
                const T2* ve = reinterpret_cast<const T2*>(&v);
#pragma unroll
                for (int u2 = 0; u2 < E / 2; ++u2) accy[tt * (E / 2) + u2] = PR::fma(qv2, ve[u2], accy[tt * (E / 2) + u2]);
              }
            }
          } else {
            racc2[h] = PR::fma(p2[jp], e, racc2[h]);
          }
          // P slot: Pi1, or the anchor G (GIN), or nothing (GMID); L slot: Lambda, or U = Lambda + rho Pi1
          const T2 pv = GI ? q2[jp] : p2[jp];
          const T2 lv = GW ? PR::fma(rho2, p2[jp], l2[jp]) : l2[jp];
          if constexpr (PAD) {
            if (MODE != GMID) *reinterpret_cast<T2*>(Ps + j * MP + 2 * i) = pv;
            if (FM == FUSED || INIT) *reinterpret_cast<T2*>(Ls + j * MP + 2 * i) = lv;
          } else {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int jj = j + u;
              if (jj < mk) {                 // packed blocks (G > 1): no tail writes
                if (MODE != GMID) Ps[jj * MP + i] = u ? pv.y : pv.x;
                if (FM == FUSED || INIT) Ls[jj * MP + i] = u ? lv.y : lv.x;
              }
            }
          }
        }
      }
      const T r2 = (racc2[0].x + racc2[1].x) + (racc2[0].y + racc2[1].y) + mkeps;
      if constexpr (XP) {
        // support-update partials of the Pi2 = (pe + eps) w_i / r that phase 2 of this iteration
        // will form (Eq.badmmc1): per member sum_j (pe_ij + eps) y_j / r_i (accumulated in the
        // sweep above) and a count of 1 per row (w_i cancels in Eq.updatex, X5)
        const T ir = (has && rowok) ? N::div(T(1), r2) : T(0);
#pragma unroll
        for (int t = 0; t < DP / 2; ++t) {
          accx[2 * t] += accy[t].x * ir;
          accx[2 * t + 1] += accy[t].y * ir;
          accy[t] = PR::make(T(0), T(0));
        }
        if (has && rowok) accm += T(1);
      }
      if constexpr (GW) {                  // a_i *= w_i / r_i: w^t_i is added by the next launch
        if (has && rowok) a.ra[k * MP + i] = rowexp - N::lg(r2);
      }
      T R = r2;
#pragma unroll
      for (int h = MP / 2; h >= 1; h >>= 1) R += __shfl_xor_sync(0xffffffffu, R, h);
      if (has && rowok) {
        const T wt = N::div(r2, R);                                      // normalised row mass
        accw += (a.rule == 1) ? sqrt(wt) : wt;
        bad |= !isfinite(wt);
      }
    }
    if constexpr (PAD && !NOSTORE) {                   // an odd m_k's last column back to its
      if (mk & 1) {                                    // single-column layout for the store
        T* const po = Ps + (mk - 1) * MP;              // (the lane wrote position 2i itself)
        T* const lo = Ls + (mk - 1) * MP;
        const T px = po[2 * i];
        const T lx = (MODE != P1ONLY) ? lo[2 * i] : T(0);
        __syncwarp();
        po[i] = px;
        if (MODE != P1ONLY) lo[i] = lx;
      }
    }
    // results leave by bulk stores from the same slots
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      const uint32_t bp = (uint32_t)(MP * cnp * (int)sizeof(T));
      if constexpr (!NOSTORE) {
        if (MODE != GMID) tma_store(dst_plan + (int64_t)MP * cp0, st, bp);
        if (MODE != P1ONLY) tma_store(a.L + (int64_t)MP * cp0, st + MP * cns, bp);
        bulk_commit();
      }
      if (nnp > 0 && nbase < 0) {    // pass t+1 did not fit beside pass t: issue it now at the ring start
        bulk_wait_read_all();
        issue(t + 1, 0, np0, nnp);
      }
    }
    if (nnp > 0 && nbase < 0) nbase = 0;
    cbase = nbase;
    cnp = nnp;
    cp0 = np0;
    cp1 = np1;
    nnp = fnp;
    np0 = fp0;
    np1 = fp1;
  }
  pdl_trigger();                                       // the consensus kernel may be scheduled
  if (lane == 0) bulk_wait_all();
  if (bad) atomicOr(a.err, ERR_NONFINITE);
  if (__any_sync(0xffffffffu, epshit) && lane == 0) atomicOr(a.err, ERR_EPSCOL);

  // this warp's partial sums of the item (segments added in a fixed butterfly order); the
  // consensus kernels add the NWARP warp partials of every item in order: no CTA barrier here
  const int64_t part = (int64_t)item * NWARP + warp;
  if constexpr (!PH2) {
    T sacc = accw;
#pragma unroll
    for (int h = MP; h < 32; h <<= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, h);
    if (seg == 0 && rowok) a.pw[part * m + i] = sacc;
  }
  if constexpr (PH2 || XP) {
    T sm_ = accm;
#pragma unroll
    for (int h = MP; h < 32; h <<= 1) sm_ += __shfl_xor_sync(0xffffffffu, sm_, h);
    T* px = a.px + (part * m + i) * (d + 1);
    if (seg == 0 && rowok) px[d] = sm_;
#pragma unroll
    for (int tt = 0; tt < DP; ++tt) {
      T sx = accx[tt];
#pragma unroll
      for (int h = MP; h < 32; h <<= 1) sx += __shfl_xor_sync(0xffffffffu, sx, h);
      if (seg == 0 && rowok && tt < d) px[tt] = sx;
    }
  }
  if constexpr (TC) {                                  // every warp's last tcgen05.ld is complete
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm_d));
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm_a));
    }
  }
}


// Row-wise cost sums for variant 2 (no C cache), one warp per sorted member -> pm[s]: lane i
// holds x_i, the member's Y rows (stride DY) are broadcast 16-byte loads, and the cost is the
// difference form sum_t (y_jt - x_it)^2 (no cancellation: the reported objective).
// P == nullptr: sum of C (Eq.rho numerator) in closed form; otherwise sum of C .* Pi1
// (surrogate objective).  Accumulated in double per member; the cluster sums are
// formed in a fixed order by k_dsum_members.
template <typename T> __host__ __device__ constexpr int cost_member_warps() { return sizeof(T) == 8 ? 2 : 4; }

template <typename T, int DP>
__global__ void __launch_bounds__(128)
k_cost_member(const int64_t* __restrict__ off, int64_t N, const int32_t* __restrict__ mem_cl,
              const T* __restrict__ Y, const T* __restrict__ x, const T* __restrict__ P,
              double* __restrict__ pm, int m, int d, int ld) {
  using V = typename Vec16<T>::type;
  using PR = Pr<T>;
  using T2 = typename PR::t;
  constexpr int E = 16 / (int)sizeof(T);
  constexpr int DY = (DP == 4) ? 4 : DP + E;
  constexpr int MKX = 32;                            // variant 2: m_k <= 32, ld <= 32
  // the member's Y rows and (objective) its Pi1 block, staged by coalesced 16-byte loads
  constexpr int NW = cost_member_warps<T>();
  __shared__ __align__(16) T sY[NW][MKX * DY];
  __shared__ __align__(16) T sP[NW][MKX * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid-stride over the sorted members (a few resident CTAs per SM instead of N / NW short
  // CTAs, whose launch and teardown bounded the kernel); x_i is reloaded only when the cluster
  // changes (members are sorted by cluster)
  T2 nx2[DP / 2], msk2[DP / 2];                      // -x_i (difference form); mask only for DP == 4
  int c_prev = -1;
  for (int64_t sidx = (int64_t)blockIdx.x * NW + warp; sidx < N; sidx += (int64_t)gridDim.x * NW) {
  const int c = mem_cl[sidx];
  const int64_t o0 = off[sidx];
  const int mk = (int)(off[sidx + 1] - o0);
  {
    const V* src = reinterpret_cast<const V*>(Y + o0 * DY);
    V* dst = reinterpret_cast<V*>(sY[warp]);
    for (int e = lane; e < mk * DY / E; e += 32) dst[e] = __ldg(src + e);
    if (P) {
      const V* ps = reinterpret_cast<const V*>(P + (int64_t)ld * o0);
      V* pd = reinterpret_cast<V*>(sP[warp]);
      for (int e = lane; e < mk * ld / E; e += 32) pd[e] = __ldcs(ps + e);
    }
  }
  const int i = lane;
  const bool rowok = i < m;
  if (c != c_prev) {
#pragma unroll
    for (int t = 0; t < DP / 2; ++t) {
      const T v0 = (rowok && 2 * t < d) ? x[((int64_t)c * m + i) * d + 2 * t] : T(0);
      const T v1 = (rowok && 2 * t + 1 < d) ? x[((int64_t)c * m + i) * d + 2 * t + 1] : T(0);
      nx2[t] = PR::make(-v0, -v1);
      msk2[t] = PR::make(2 * t < d ? T(1) : T(0), 2 * t + 1 < d ? T(1) : T(0));
    }
    c_prev = c;
  }
  __syncwarp();
  if (!P) {
    // Eq.rho numerator in closed form, in fp64 (products of fp32 values are exact there):
    //   sum_ij |x_i - y_j|^2 = m_k sum_i |x_i|^2 + m sum_j |y_j|^2 - 2 sum_i x_i . (sum_j y_j)
    // O((m + m_k) d) per member instead of O(m m_k d); the cancellation costs no more than a few
    // digits of fp64 (|x|^2, |y|^2 within a small factor of the cost on these workloads)
    __shared__ double sSy[NW][16];
    double q = 0.0;                                   // lane t < d: sum_j y_jt^2, then sum_j y_jt
    if (lane < d && lane < 16) {
      double sy = 0.0;
      for (int j = 0; j < mk; ++j) {
        const double v = (double)sY[warp][j * DY + lane];
        sy += v;
        q = fma(v, v, q);
      }
      sSy[warp][lane] = sy;
    }
    __syncwarp();
    double xi2 = 0.0, xdot = 0.0;                     // lane i < m: |x_i|^2 and x_i . sum_j y_j
#pragma unroll
    for (int t = 0; t < DP / 2; ++t) {                // nx2 = -x_i (0 past d and for rows >= m)
      const double x0 = -(double)nx2[t].x, x1 = -(double)nx2[t].y;
      xi2 = fma(x0, x0, fma(x1, x1, xi2));
      if (2 * t < d) xdot = fma(x0, sSy[warp][2 * t], xdot);
      if (2 * t + 1 < d) xdot = fma(x1, sSy[warp][2 * t + 1], xdot);
    }
    double acc = (double)mk * xi2 - 2.0 * xdot + (double)m * q;
    for (int h = 16; h >= 1; h >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, h);
    if (lane == 0) pm[sidx] = acc;
    __syncwarp();                                   // sY / sSy reused by the next member
    continue;
  }
  T s = T(0);
  for (int j0 = 0; j0 < mk; j0 += 4) {
    T2 c2[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = (j0 + u < mk) ? j0 + u : mk - 1;
      const T* yj = sY[warp] + j * DY;
      c2[u] = PR::make(T(0), T(0));
#pragma unroll
      for (int tt = 0; tt < DP / E; ++tt) {
        const V v = *reinterpret_cast<const V*>(yj + tt * E);
#pragma unroll
        for (int u2 = 0; u2 < E / 2; ++u2) {
          const T2 yv = reinterpret_cast<const T2*>(&v)[u2];
          // y - x on the real coordinates: for DP >= 16 the slots [d, DP) of a Y row are 0 (and
          // |y|^2 sits at DP), for DP == 4 the |y|^2 slot is inside the row and is masked
          T2 df = PR::add(yv, nx2[tt * (E / 2) + u2]);
          if constexpr (DP == 4) df = PR::mul(df, msk2[tt * (E / 2) + u2]);
          c2[u] = PR::fma(df, df, c2[u]);
        }
      }
    }
    // Pi1 of the four columns (pair layout for 32-row blocks: one 8-byte read per column pair,
    // conflict-free; an odd m_k's last column single)
    T pv[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = j0 + 2 * h;
      if (ld == 32 && j + 1 < mk) {
        const T2 q = *reinterpret_cast<const T2*>(&sP[warp][j * ld + 2 * i]);
        pv[2 * h] = q.x;
        pv[2 * h + 1] = q.y;
      } else {
        pv[2 * h] = j < mk ? sP[warp][j * ld + i] : T(0);
        pv[2 * h + 1] = j + 1 < mk ? sP[warp][(j + 1) * ld + i] : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j0 + u < mk && rowok) s += (c2[u].x + c2[u].y) * pv[u];
  }
  double acc = (double)s;
  for (int h = 16; h >= 1; h >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, h);
  if (lane == 0) pm[sidx] = acc;
  __syncwarp();
  }
}

}  // namespace ad2k
