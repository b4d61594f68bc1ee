// ad2_wide.cuh — fused B-ADMM iteration kernel for 32 < m <= 64 (variant 3, fp32): a warp PAIR
// per member.  Modified B-ADMM of AD2-clustering (arXiv 1510.00012, Alg. 4).
//
// Member blocks have WM = 64 (or 32, one warp per member) rows (ld = WM, rows >= m zero) and
// m_k <= MKX (64 or 128) columns.  Lane i of warp h of a group owns centroid row 32h + i for EVERY
// column of the member, so row sums are lane-local.  The state does not live in registers (a 64-column row would need ~200): the pass
// region [P | L | C] of one member is staged by three cp.async.bulk loads into a per-pair ring and
// the iteration is three column sweeps over shared memory (each entry's intermediate is written
// back in place), plus a column-sum step in which lane j of the pair reads column j's 64 rows
// (16 rotated 16-byte loads, bank-conflict free).  C is the cached cost (d up to 64 makes
// recomputing it per iteration as expensive as reading it), so an iteration
// moves 20 B per entry: P, L in and out, C in.
//
//   MODE P1ONLY: Pi2 (= Q) -> sweep B (Eq.badmmc0b) -> column sums -> sweep C (Eq.badmmc0, the
//                Eq.badmmc1b row masses) -> P = Pi1, w-partials
//   MODE FUSED : sweep A (Eq.badmmc1b with Lambda^n, row mass, Lambda + rho Pi1) -> sweep B
//                (Eq.badmmc1 with the consensus w, Eq.badmm2, then Eq.badmmc0b) -> column sums ->
//                sweep C -> P = Pi1, L = Lambda, w-partials
//   MODE P2ONLY: sweep A -> sweep B2 (Eq.badmmc1, Eq.badmm2, support-update partials of
//                Eq.updatex) -> Q = Pi2, L = Lambda, x-partials
//   MODE P2X   : P2ONLY without the stores (the x partials only): the step's phase 2 stays deferred
//                and the next step's first FUSED pass recomputes it (it reads no cost)
//   MODE P1INIT: P1ONLY of a cold round with Pi2^0 = w_i w_j^(k) and Lambda = 0 formed in the sweep
//                (only C is loaded; L = 0 is stored with Pi1): no k_init_plans pass
//   MODE FUSEDX: FUSED + a sweep D forming the support-update partials of the Pi2 that the deferred
//                phase 2 will produce, (pe + eps) / r2 with pe = Pi1 exp(Lambda/rho) (w_i cancels in
//                Eq.updatex): the last pass of a step of n >= 2 iterations, so no P2 pass
#pragma once
#include "ad2_tma.cuh"

#ifndef AD2_WIDE_XMMA
#define AD2_WIDE_XMMA 1
#endif

namespace ad2k {

// WM = rows of a member block (ld) = 32 x warps per member group; MKX = largest m_k; NPAIR groups
// per CTA, each with a ring of RING_KB
template <int WM, int MKX, int NPAIR, int RING_KB>
struct WideLayout {
  static constexpr int RING = RING_KB * 1024 / 4;               // floats per group
  // [ring | fbuf[MKX] | Rw[4] | Rr[WM] | 3 mbarriers (load pipeline; FUSEDX: the supports into the C slot)]
  static constexpr size_t PAIR_BYTES = ((4 * (size_t)(RING + MKX + 4 + WM) + 24) + 127) / 128 * 128;   // + 3 mbarriers
  static constexpr size_t CTA_BYTES = NPAIR * PAIR_BYTES;
  static_assert(RING >= 3 * WM * MKX, "ring must hold the largest pass");
  static_assert(CTA_BYTES <= 227 * 1024, "shared memory");
};

template <int WM>
__device__ __forceinline__ void group_sync(int id) {
  if constexpr (WM == 128) asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
  else if constexpr (WM == 64) asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
  else __syncwarp();
}

// 3 x TF32 on the warp-level tensor-core MMA (mma.sync m16n8k8, fp32 accumulate): v = hi + lo with
// hi = tf32(v), lo = tf32(v - hi); a.b ~ a_hi b_hi + a_hi b_lo + a_lo b_hi (a_lo b_lo ~ 2^-22 dropped)
__device__ __forceinline__ void tf32_split(float v, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(v));
  const float r = v - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}
__device__ __forceinline__ void mma_tf32(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int WM, int MKX, int NPAIR, int RING_KB, int MODE, int DP>
__global__ void __launch_bounds__(NPAIR * WM, 1)
k_badmm_wide(const IterArgs<float> a) {
  constexpr int WMP = WM;
  constexpr int WMK = MKX;
  constexpr int GW = WM / 32;                                      // warps per member group
  using Lay = WideLayout<WM, MKX, NPAIR, RING_KB>;
  using N = Num<float>;
  constexpr int RING = Lay::RING;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp / GW, h = warp % GW;
  float* const ring = reinterpret_cast<float*>(smem_raw + (size_t)pair * Lay::PAIR_BYTES);
  float* const fbuf = ring + RING;                                 // Eq.badmmc0 column factors
  float* const Rw = fbuf + WMK;                                    // per-warp row-mass totals
  float* const Rr = Rw + 4;                                        // FUSEDX: 1 / row mass of every row
  uint64_t* const bar = reinterpret_cast<uint64_t*>(Rr + WM);
  const bool leader = (h == 0 && lane == 0);
  const int bar_id = 1 + pair;
  const int ig = 32 * h + lane;                                    // this lane's centroid row
  const int item = a.perm ? a.perm[blockIdx.x] : (int)blockIdx.x;
  const int c = a.item_cl[item];
  const int64_t mb = a.item_mb[item], me = a.item_mb[item + 1];
  const int m = a.m, d = a.d;
  const bool rowok = ig < m;
  const float kx = a.kx[c], rho = a.rho[c];
  const float eps_r = rowok ? a.eps : 0.f;
  const float wi = (MODE != P1ONLY && rowok) ? a.w[(int64_t)c * m + ig] : 0.f;
  // Lambda pre-scaled: L' = Lambda kx (kx = log2(e)/rho), dual step kappa = kx rho = log2(e)
  (void)rho;
  const float kap = N::kappa();
  const float2 nkx2 = make_float2(-kx, -kx);
  const float2 rho2 = make_float2(kap, kap), nrho2 = make_float2(-kap, -kap);
  const float2 eps2 = make_float2(eps_r, eps_r);
  float accw = 0.f, accm = 0.f;
  constexpr bool PH2 = (MODE == P2ONLY || MODE == P2X);
  constexpr bool XP = (MODE == FUSEDX);                            // FUSED + the support-update partials
  constexpr bool INIT = (MODE == P1INIT);                          // cold round's first pass: Pi2^0 = w_i w_j^(k), Lambda = 0
  constexpr bool PH1 = (MODE == P1ONLY || INIT);
  constexpr int FM = XP ? FUSED : MODE;                            // the mode the sweeps follow
  float2 accx[(PH2 || XP) ? DP / 2 : 1];                           // coordinate pairs (FFMA2)
  // FUSEDX of the 64-row pair with d <= 64: the partials on the tensor cores (3 x TF32 mma.sync)
  constexpr bool XMMA = XP && WM == 64 && DP == 64 && AD2_WIDE_XMMA;
  float* const xacc = reinterpret_cast<float*>(accx);            // XMMA: [2 row tiles][8 col tiles][4]
#pragma unroll
  for (int t = 0; t < ((PH2 || XP) ? DP / 2 : 1); ++t) accx[t] = make_float2(0.f, 0.f);
  bool bad = false;
  const float* src_plan = (MODE == P1ONLY) ? a.Q : a.P;
  float* dst_plan = (MODE == P2ONLY) ? a.Q : a.P;

  if (leader) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    if constexpr (MODE == FUSEDX) mbar_init(&bar[2], 1);
    fence_mbar_init();
  }
  group_sync<WM>(bar_id);

  auto member = [&](int t, int64_t& p0) -> int {                  // pair-uniform
    const int64_t k = mb + pair + (int64_t)t * NPAIR;
    if (k >= me) return 0;
    p0 = a.off[k];
    return (int)(a.off[k + 1] - p0);
  };
  // pass region [P | L | C] (P2ONLY: [P | L | Y], the supports for the x partials); dy % 4 == 0
  const int dy = a.dy;
  // P2ONLY with external x partials (d > 64, k_xpart) stages no supports
  const int third = PH2 ? (a.xext ? 0 : dy) : WMP;                 // floats per point of the 3rd array
  auto issue = [&](int t, int base, int64_t p0, int np) {          // leader only
    const uint32_t bp = (uint32_t)(WMP * np * 4), b3 = (uint32_t)(third * np * 4);
    float* st = ring + base;
    mbar_expect_tx(&bar[t & 1], INIT ? b3 : 2 * bp + b3);
    if (!INIT) {                                                   // P1INIT forms P and L itself
      tma_load(st, src_plan + (int64_t)WMP * p0, bp, &bar[t & 1]);
      tma_load(st + WMP * np, a.L + (int64_t)WMP * p0, bp, &bar[t & 1]);
    }
    if (PH2) {
      if (b3) tma_load(st + 2 * WMP * np, a.Y + (int64_t)dy * p0, b3, &bar[t & 1]);
    }
    else tma_load(st + 2 * WMP * np, a.Cc + (int64_t)WMP * p0, b3, &bar[t & 1]);
  };

  int64_t cp0 = 0;
  int cnp = member(0, cp0);
  int cbase = 0;
  if (leader && cnp > 0) issue(0, 0, cp0, cnp);
  int64_t np0 = 0;                                 // geometry of pass t+1, loaded one pass ahead
  int nnp = member(1, np0);

  for (int t = 0; cnp > 0; ++t) {
    // place pass t+1 beside pass t (alternating ring start / ring end) while t computes
    int64_t fp0 = 0;
    const int fnp = member(t + 2, fp0);            // consumed next pass
    const int csize = (2 * WMP + third) * cnp, nsize = (2 * WMP + third) * nnp;
    int nbase = -1;
    if (nnp > 0) {
      if (cbase == 0) {
        if (RING - nsize >= csize) nbase = RING - nsize;
      } else if (nsize <= cbase) {
        nbase = 0;
      }
    }
    AD2_CHECK(cnp <= MKX && nnp <= MKX && cbase >= 0 && cbase + csize <= RING);
    AD2_CHECK(nbase < 0 || (nbase + nsize <= RING && (nbase >= cbase + csize || nbase + nsize <= cbase)));
    if (leader && nbase >= 0) {
      bulk_wait_read_all();            // pass t-1 has left its region
      issue(t + 1, nbase, np0, nnp);
    }
    const int mk = cnp;
    const int jc = ig;                 // the column this lane sums (jc < mk)
    float om_jc[(MKX + WM - 1) / WM];               // w^(k)_j of the columns this lane sums
#pragma unroll
    for (int cj = 0; cj < (MKX + WM - 1) / WM; ++cj)
      om_jc[cj] = (!PH2 && jc + cj * WM < mk) ? __ldg(a.om + cp0 + jc + cj * WM) : 0.f;
    mbar_wait(&bar[t & 1], (uint32_t)((t >> 1) & 1));
    float* const Ps = ring + cbase;
    float* const Ls = Ps + WMP * mk;
    const float* const Cs = Ls + WMP * mk;                         // C (P2ONLY: Y rows, stride dy)

    // ---- sweep A (phase 2 of iteration t-1): row mass r = sum_j Pi1 exp(Lambda/rho) + m_k eps
    //      (Eq.badmmc1b; Lambda is stored pre-scaled, L' = Lambda kx, so exp(Lambda/rho) = ex(L'))
    float f = 0.f;
    if constexpr (!PH1) {
      float2 racc = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int j = 0; j < mk; j += 2) {
        const bool v1 = j + 1 < mk;
        const int e0 = j * WMP + ig, e1 = e0 + WMP;
        const float2 p = make_float2(Ps[e0], v1 ? Ps[e1] : 0.f);
        const float2 l = make_float2(Ls[e0], v1 ? Ls[e1] : 0.f);
        racc = __ffma2_rn(p, make_float2(N::ex(l.x), N::ex(l.y)), racc);
      }
      const float r = (racc.x + racc.y) + (float)mk * eps_r;
      f = rowok ? __fdividef(wi, r) : 0.f;                           // Eq.badmmc1: w_i / row mass
    }
    const float2 f2 = make_float2(f, f), ef2 = make_float2(eps_r * f, eps_r * f);

    if constexpr (PH2) {
      // ---- sweep B2: Pi2 = (pe + eps) w_i / r (Eq.badmmc1), L' += kappa (Pi1 - Pi2) (Eq.badmm2),
      //      support-update partials sum_j pi2_ij y_j, sum_j pi2_ij (Eq.updatex, X5)
#pragma unroll 2
      for (int j = 0; j < mk; ++j) {
        const int e0 = j * WMP + ig;
        const float p = Ps[e0], l = Ls[e0];
        const float q = fmaf(p * N::ex(l), f, eps_r * f);
        const float2 q2 = make_float2(q, q);
        if constexpr (MODE == P2ONLY) {
          Ps[e0] = q;
          Ls[e0] = fmaf(-kap, q, fmaf(kap, p, l));
        }
        if (a.xext) continue;
        accm += q;
        const float* yj = Cs + j * dy;
#pragma unroll
        for (int tt = 0; tt < DP / 4; ++tt) {
          if (4 * tt < d) {
            const float4 v = *(reinterpret_cast<const float4*>(yj) + tt);
            accx[2 * tt + 0] = __ffma2_rn(q2, make_float2(v.x, v.y), accx[2 * tt + 0]);
            accx[2 * tt + 1] = __ffma2_rn(q2, make_float2(v.z, v.w), accx[2 * tt + 1]);
          }
        }
      }
      fence_proxy_async_smem();
      group_sync<WM>(bar_id);
    } else {
      // ---- sweep B: (FUSED) Pi2 = (Pi1 exp(Lambda/rho) + eps) f (Eq.badmmc1, pe recomputed),
      //      L' += kappa (Pi1 - Pi2) (Eq.badmm2); pt2 = Pi2 exp(-(C + Lambda)/rho) + eps
      //      (Eq.badmmc0b) = Pi2 ex(-(C kx + L')) + eps -> Ps
      if constexpr (INIT) {                                            // w^(k)_j for sweep B (fbuf is free)
#pragma unroll
        for (int cj = 0; cj < (MKX + WM - 1) / WM; ++cj)
          if (jc + cj * WM < mk) fbuf[jc + cj * WM] = om_jc[cj];
        group_sync<WM>(bar_id);
      }
#pragma unroll 4
      for (int j = 0; j < mk; j += 2) {
        const bool v1 = j + 1 < mk;
        const int e0 = j * WMP + ig, e1 = e0 + WMP;
        // P1INIT: Pi2^0 = w_i w_j^(k), Lambda = 0; else Pi1 / Pi2 and Lambda from the slots
        const float2 p = INIT ? make_float2(wi * fbuf[j], v1 ? wi * fbuf[j + 1] : 0.f)
                              : make_float2(Ps[e0], v1 ? Ps[e1] : 0.f);
        float2 l = INIT ? make_float2(0.f, 0.f) : make_float2(Ls[e0], v1 ? Ls[e1] : 0.f);
        const float2 cst = make_float2(Cs[e0], v1 ? Cs[e1] : 0.f);
        float2 q = p;                                                  // P1ONLY: Pi2^(0)
        if constexpr (FM == FUSED) {
          q = __ffma2_rn(__fmul2_rn(p, make_float2(N::ex(l.x), N::ex(l.y))), f2, ef2);
          l = __ffma2_rn(nrho2, q, __ffma2_rn(rho2, p, l));
        }
        const float2 ar = __ffma2_rn(cst, nkx2, make_float2(-l.x, -l.y));
        const float2 pt = __ffma2_rn(q, make_float2(N::ex(ar.x), N::ex(ar.y)), eps2);
        Ps[e0] = pt.x;
        if (FM == FUSED || INIT) Ls[e0] = l.x;
        if (v1) {
          Ps[e1] = pt.y;
          if (FM == FUSED || INIT) Ls[e1] = l.y;
        }
      }
      if constexpr (XP) fence_proxy_async_smem();                       // the C slot's reads -> the async write below
      group_sync<WM>(bar_id);
      if constexpr (XP) {
        // C is consumed: the member's support rows (dy <= WM floats each) come into the C slot while
        // the column sums and sweep C run, for sweep D below
        if (leader) {
          const uint32_t by = (uint32_t)(dy * mk * 4);
          mbar_expect_tx(&bar[2], by);
          tma_load(const_cast<float*>(Cs), a.Y + (int64_t)dy * cp0, by, &bar[2]);
        }
      }
      // ---- column sums over the 64 rows (Eq.badmmc0 denominators): lane jc reads its column in
      //      16 chunks of 4 rows, starting at chunk jc mod 16 (4 lanes per bank quad: no conflicts)
#pragma unroll
      for (int cj = 0; cj < (WMK + WM - 1) / WM; ++cj) {               // WM = 32: two columns per lane
        const int jcc = jc + cj * WM;
        if (jcc < mk) {
          const float* col = Ps + jcc * WMP;
          float2 s0 = make_float2(0.f, 0.f), s1 = make_float2(0.f, 0.f);
#pragma unroll
          for (int u = 0; u < WM / 4; ++u) {
            const int chn = (u + jcc) & (WM / 4 - 1);
            const float4 v = *reinterpret_cast<const float4*>(col + 4 * chn);
            s0 = __fadd2_rn(s0, make_float2(v.x, v.y));
            s1 = __fadd2_rn(s1, make_float2(v.z, v.w));
          }
          const float s = (s0.x + s0.y) + (s1.x + s1.y);
          fbuf[jcc] = __fdividef(om_jc[cj], s);                          // Eq.badmmc0: w_j^(k) / colsum
        }
      }
      group_sync<WM>(bar_id);
      // ---- sweep C: Pi1 = pt2 * factor_j -> Ps; pt1 = Pi1 exp(Lambda/rho) + eps (Eq.badmmc1b) row mass
      float2 racc = make_float2(0.f, 0.f);
#pragma unroll 4
      for (int j = 0; j < mk; j += 2) {
        const bool v1 = j + 1 < mk;
        const int e0 = j * WMP + ig, e1 = e0 + WMP;
        const float2 pt = make_float2(Ps[e0], v1 ? Ps[e1] : 0.f);
        const float2 l = make_float2(Ls[e0], v1 ? Ls[e1] : 0.f);
        const float2 fj = make_float2(fbuf[j], v1 ? fbuf[j + 1] : 0.f);
        const float2 p1 = __fmul2_rn(pt, fj);
        racc = __ffma2_rn(p1, make_float2(N::ex(l.x), N::ex(l.y)), racc);
        Ps[e0] = p1.x;
        if (v1) Ps[e1] = p1.y;
      }
      const float r2 = (racc.x + racc.y) + (float)mk * eps_r;
      if constexpr (XP) Rr[ig] = rowok ? __fdividef(1.f, r2) : 0.f;   // for sweep D (group-synced below)
      float R = r2;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) R += __shfl_xor_sync(0xffffffffu, R, o);
      fence_proxy_async_smem();
      if constexpr (WM >= 64) {
        if (lane == 0) Rw[h] = R;
        group_sync<WM>(bar_id);
        R = (WM == 128) ? (Rw[0] + Rw[1]) + (Rw[2] + Rw[3]) : Rw[0] + Rw[1];
      } else {
        __syncwarp();
      }
      if (rowok) {
        const float wt = __fdividef(r2, R);                            // normalised row mass
        accw += (a.rule == 1) ? sqrtf(wt) : wt;
        bad |= !isfinite(wt);
      }
      if constexpr (XP) {
        // support-update partials of the Pi2 = (pe + eps) w_i / r2 that phase 2 of this iteration
        // will form (Eq.badmmc1; w_i cancels in Eq.updatex, X5): per row sum_j (pe_ij + eps) y_j / r2
        // and a count of 1, pe = Pi1 exp(Lambda/rho) re-read from the slots.  Warp h of the group
        // forms coordinates [h TS, (h + 1) TS) for every row 32 g + lane (g < GW), so each broadcast
        // 16-byte load of a support row (four quarter-warp wavefronts) feeds GW rows; per (row,
        // coordinate) the sum over j has the same order as with one row per lane (bit-identical)
        if constexpr (XMMA) {
          // X_part[r][t] += sum_j q_rj y_jt on the tensor cores: warp h owns rows [32h, 32h + 32)
          // (two 16-row tiles) x 64 coordinates (eight 8-column tiles), K = the member's points in
          // steps of 8; the A fragments q_rj are formed in place from the P / L slots, the B
          // fragments are the support rows in the C slot (points >= m_k: q = 0 and y = 0)
          const int gid = lane >> 2, tig = lane & 3;
          float irr[2][2], epr[2][2];
#pragma unroll
          for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) {
              const int r = 32 * h + 16 * mt + gid + 8 * hr;
              irr[mt][hr] = Rr[r];
              epr[mt][hr] = r < m ? a.eps : 0.f;
            }
          mbar_wait(&bar[2], (uint32_t)(t & 1));
          for (int k0 = 0; k0 < mk; k0 += 8) {
            uint32_t ah[2][4], al[2][4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
              for (int e = 0; e < 4; ++e) {            // a0 (gid, tig) a1 (gid+8, tig) a2 (gid, tig+4) a3 (gid+8, tig+4)
                const int hr = e & 1, j = k0 + tig + 4 * (e >> 1);
                const int r = 32 * h + 16 * mt + gid + 8 * hr;
                float q = 0.f;
                if (j < mk) {
                  const int e0 = j * WMP + r;
                  q = fmaf(Ps[e0], N::ex(Ls[e0]), epr[mt][hr]) * irr[mt][hr];
                }
                tf32_split(q, ah[mt][e], al[mt][e]);
              }
            const int j0 = k0 + tig, j1 = j0 + 4;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
              const int tc = 8 * nt + gid;
              const float y0 = (j0 < mk && tc < dy) ? Cs[j0 * dy + tc] : 0.f;
              const float y1 = (j1 < mk && tc < dy) ? Cs[j1 * dy + tc] : 0.f;
              uint32_t bh0, bl0, bh1, bl1;
              tf32_split(y0, bh0, bl0);
              tf32_split(y1, bh1, bl1);
#pragma unroll
              for (int mt = 0; mt < 2; ++mt) {
                float* acc = xacc + (mt * 8 + nt) * 4;
                mma_tf32(acc, ah[mt], bh0, bh1);
                mma_tf32(acc, ah[mt], bl0, bl1);
                mma_tf32(acc, al[mt], bh0, bh1);
              }
            }
          }
          accm += 1.f;
          fence_proxy_async_smem();
          group_sync<WM>(bar_id);
        } else {
        constexpr int TS = DP / GW;
        const int t0 = h * TS;
        float irg[GW], epsg[GW];
#pragma unroll
        for (int g = 0; g < GW; ++g) {
          irg[g] = Rr[32 * g + lane];
          epsg[g] = (32 * g + lane < m) ? a.eps : 0.f;
        }
        mbar_wait(&bar[2], (uint32_t)(t & 1));
#pragma unroll 2
        for (int j = 0; j < mk; ++j) {
          float q[GW];
#pragma unroll
          for (int g = 0; g < GW; ++g) {
            const int e0 = j * WMP + 32 * g + lane;
            q[g] = fmaf(Ps[e0], N::ex(Ls[e0]), epsg[g]) * irg[g];
          }
          const float4* yj = reinterpret_cast<const float4*>(Cs + j * dy + t0);
#pragma unroll
          for (int tt = 0; tt < TS / 4; ++tt) {
            if (t0 + 4 * tt < d) {
              const float4 v = yj[tt];
#pragma unroll
              for (int g = 0; g < GW; ++g) {
                const float2 q2 = make_float2(q[g], q[g]);
                float2& a0 = accx[g * (TS / 2) + 2 * tt + 0];
                float2& a1 = accx[g * (TS / 2) + 2 * tt + 1];
                a0 = __ffma2_rn(q2, make_float2(v.x, v.y), a0);
                a1 = __ffma2_rn(q2, make_float2(v.z, v.w), a1);
              }
            }
          }
        }
        accm += 1.f;                                   // member passes (rows >= m are never written)
        // the group's reads of the slot are done before the leader may load the next pass over it
        fence_proxy_async_smem();
        group_sync<WM>(bar_id);
        }
      }
    }
    // ---- results leave by bulk stores from the same slots
    if (leader) {
      const uint32_t bp = (uint32_t)(WMP * mk * 4);
      if (MODE != P2X) {
        tma_store(dst_plan + (int64_t)WMP * cp0, Ps, bp);
        if (MODE != P1ONLY) tma_store(a.L + (int64_t)WMP * cp0, Ls, bp);
        bulk_commit();
      }
      if (nnp > 0 && nbase < 0) {      // pass t+1 did not fit beside pass t: issue it at the ring start
        bulk_wait_read_all();
        issue(t + 1, 0, np0, nnp);
      }
    }
    if (nnp > 0 && nbase < 0) nbase = 0;
    cbase = nbase;
    cnp = nnp;
    cp0 = np0;
    nnp = fnp;
    np0 = fp0;
  }
  if (leader) bulk_wait_all();
  if (bad) atomicOr(a.err, ERR_NONFINITE);

  // this pair's partial sums of the item (rows are lane-owned); consensus adds the NPAIR pair
  // partials of every item in order
  const int64_t part = (int64_t)item * NPAIR + pair;
  if constexpr (!PH2) {
    if (rowok) a.pw[part * m + ig] = accw;
  }
  if constexpr (PH2) {
    if (rowok && !a.xext) {
      float* px = a.px + (part * m + ig) * (d + 1);
      px[d] = accm;
#pragma unroll
      for (int t = 0; t < DP; ++t)
        if (t < d) px[t] = (t & 1) ? accx[t / 2].y : accx[t / 2].x;
    }
  }
  if constexpr (XMMA) {                                // C fragments: (gid, 2tig), (gid, 2tig+1), (gid+8, ..)
    const int gid = lane >> 2, tig = lane & 3;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int row = 32 * h + 16 * mt + gid + 8 * hr;
        if (row < m) {
          float* px = a.px + (part * m + row) * (d + 1);
#pragma unroll
          for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int tc = 8 * nt + 2 * tig + e;
              if (tc < d) px[tc] = xacc[(mt * 8 + nt) * 4 + 2 * hr + e];
            }
        }
      }
    if (32 * h + lane < m) a.px[(part * m + 32 * h + lane) * (d + 1) + d] = accm;
  } else if constexpr (XP) {                           // warp h: coordinates [h TS, (h + 1) TS) of every row
    constexpr int TS = DP / GW;
#pragma unroll
    for (int g = 0; g < GW; ++g) {
      const int row = 32 * g + lane;
      if (row < m) {
        float* px = a.px + (part * m + row) * (d + 1);
        if (h == 0) px[d] = accm;
#pragma unroll
        for (int u = 0; u < TS; ++u) {
          const int tc = h * TS + u;
          if (tc < d) px[tc] = (u & 1) ? accx[g * (TS / 2) + u / 2].y : accx[g * (TS / 2) + u / 2].x;
        }
      }
    }
  }
}

// Cost build for the cached-C variants: C_ij = |x_i|^2 + |y_j|^2 - 2 x_i.y_j in fp32,
// clamped at 0, for a 64 x 64 (rows x points) tile per step: X_c^T (coordinate-major) stays in
// shared memory per row block; the points come in chunks of 64 rows (row-major, 16-byte cp.async,
// coalesced) into two buffers, the next chunk landing while the current one computes; each thread
// accumulates a 4 x 4 register tile of dot products over t = 0..d-1 in order (per 4 coordinates:
// four 16-byte x loads of 4 rows, four broadcast 16-byte y loads of 4 points, 32 FFMA2).
// Entries of rows >= m are written as 0.  With psum != nullptr the per-item double sum of C
// (Eq.rho numerator) is formed in a fixed order.  One CTA (256 threads) per work item.
template <int DMAX>
struct CostTile {
  static constexpr int YP = DMAX + 4;                  // row pitch of a staged point (floats)
  static constexpr size_t XS = sizeof(float) * DMAX * 68;
  static constexpr size_t YS = sizeof(float) * 64 * YP;
  static constexpr size_t BYTES = XS + 2 * YS + sizeof(float) * (64 + 2 * 64);
};

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(sdst)),
               "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int DMAX>
__global__ void __launch_bounds__(256)
k_cost_tile(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
            const int32_t* __restrict__ item_cl, const float* __restrict__ Y, const float* __restrict__ x,
            float* __restrict__ Cc, double* __restrict__ psum, int m, int d, int dy, int ld) {
  using L = CostTile<DMAX>;
  constexpr int YP = L::YP;
  extern __shared__ __align__(16) unsigned char ct_smem[];
  float (*xs)[68] = reinterpret_cast<float (*)[68]>(ct_smem);                  // [DMAX][68]
  float (*ysb)[64][YP] = reinterpret_cast<float (*)[64][YP]>(ct_smem + L::XS);  // [2][64][YP]
  float* xx = reinterpret_cast<float*>(ct_smem + L::XS + 2 * L::YS);           // [64]
  float* yyb = xx + 64;                                                        // [2][64]
  __shared__ double red[8];
  const int item = blockIdx.x;
  const int c = item_cl[item];
  const int tid = threadIdx.x;
  const int ti = tid & 15, tj = tid >> 4;              // rows 4ti..4ti+3, points 4tj..4tj+3
  const int64_t p_beg = off[item_mb[item]], p_end = off[item_mb[item + 1]];
  const int dpad = (d + 3) & ~3;                       // Y rows are zero-padded to dpad (= dy)
  const int pieces = dpad >> 2;
  auto load_chunk = [&](int buf, int64_t q0) {
    const int np = (int)((p_end - q0) < 64 ? (p_end - q0) : 64);
    for (int v = tid; v < np * pieces; v += 256) {
      const int j = v / pieces, k = v - j * pieces;
      cp_async16(&ysb[buf][j][4 * k], Y + (q0 + j) * dy + 4 * k);
    }
    cp_async_commit();
  };
  double acc = 0.0;
  for (int rb = 0; rb < ld; rb += 64) {                // row blocks of 64 (ld = 128 for m > 64)
    __syncthreads();                                   // the previous row block's buffers are free
    if (p_beg < p_end) load_chunk(0, p_beg);
    for (int v = tid; v < DMAX * 64; v += 256) {
      const int t = v >> 6, i = v & 63;
      xs[t][i] = (rb + i < m && t < d) ? x[((int64_t)c * m + rb + i) * d + t] : 0.f;
    }
    __syncthreads();
    if (tid < 64) {
      float s = 0.f;
      for (int t = 0; t < d; ++t) s = fmaf(xs[t][tid], xs[t][tid], s);
      xx[tid] = s;
    }
    int buf = 0;
    for (int64_t q0 = p_beg; q0 < p_end; q0 += 64, buf ^= 1) {
      const int np = (int)((p_end - q0) < 64 ? (p_end - q0) : 64);
      if (q0 + 64 < p_end) {                           // the next chunk lands while this one computes
        load_chunk(buf ^ 1, q0 + 64);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();                                 // chunk `buf` visible to every thread
      float (*ys)[YP] = ysb[buf];
      float* yy = yyb + 64 * buf;
      if (tid < 64) {
        float s = 0.f;
        for (int t = 0; t < d; ++t) s = fmaf(ys[tid][t], ys[tid][t], s);
        yy[tid] = s;
      }
      float2 a2[2][4];                                 // rows (4ti, 4ti+1) and (4ti+2, 4ti+3) x 4 points
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) a2[u][v] = make_float2(0.f, 0.f);
#pragma unroll 2
      for (int t = 0; t < dpad; t += 4) {
        float4 y4[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) y4[v] = *reinterpret_cast<const float4*>(&ys[4 * tj + v][t]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 xv = *reinterpret_cast<const float4*>(&xs[t + k][4 * ti]);
          const float2 x01 = make_float2(xv.x, xv.y), x23 = make_float2(xv.z, xv.w);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const float yk = k == 0 ? y4[v].x : (k == 1 ? y4[v].y : (k == 2 ? y4[v].z : y4[v].w));
            const float2 yy2 = make_float2(yk, yk);
            a2[0][v] = __ffma2_rn(x01, yy2, a2[0][v]);
            a2[1][v] = __ffma2_rn(x23, yy2, a2[1][v]);
          }
        }
      }
      __syncthreads();                                 // yy ready; every read of ys[buf] done
      float s = 0.f;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int j = 4 * tj + v;
        if (j < np && rb + 4 * ti < ld) {
          float4 o;
          float* oe = reinterpret_cast<float*>(&o);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = rb + 4 * ti + u;
            const float dot = (u & 1) ? a2[u >> 1][v].y : a2[u >> 1][v].x;
            const float cv = (i < m) ? fmaxf(fmaf(-2.f, dot, xx[i - rb] + yy[j]), 0.f) : 0.f;
            oe[u] = cv;
            s += cv;
          }
          *reinterpret_cast<float4*>(Cc + (q0 + j) * ld + rb + 4 * ti) = o;
        }
      }
      acc += (double)s;
    }
  }
  if (psum) {
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      psum[item] = t;
    }
  }
}

// The same build with 8 x 8 register tiles (16 < d <= 64, the default): a CTA of 128 threads
// computes a 64-row x 128-point tile per chunk, thread (ti, tj) owning rows {4ti..4ti+3,
// 32+4ti..32+4ti+3} and points {4tj..4tj+3, 64+4tj..64+4tj+3}; per 4 coordinates 8 + 8 16-byte
// loads feed 128 FFMA2 (0.25 shared-memory wavefront per FMA instead of 0.5).  One point buffer
// (the next chunk's cp.async is issued after the last read of the current one and lands during the
// epilogue) so 4 CTAs fit per SM (124 registers): measured on config 4 (ncu, cold) 4.17 ms per
// build vs 4.93 (4 x 4 tiles), 4.43 at 3 CTAs per SM, 5.40 with two buffers at 2 CTAs per SM.
// Same dot-product order (t = 0..d-1) and the same |x|^2, |y|^2 chains: C is bit-identical to
// k_cost_tile's (the per-item rho sums differ in order).
struct CostTile8 {
  static constexpr int YP = 68;
  static constexpr size_t XS = sizeof(float) * 64 * 68;
  static constexpr size_t YS = sizeof(float) * 128 * YP;
  static constexpr size_t BYTES = XS + YS + sizeof(float) * (64 + 2 * 128);
};

__global__ void __launch_bounds__(128, 4)
k_cost_tile8(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
             const int32_t* __restrict__ item_cl, const float* __restrict__ Y, const float* __restrict__ x,
             float* __restrict__ Cc, double* __restrict__ psum, int m, int d, int dy, int ld) {
  using L = CostTile8;
  constexpr int YP = L::YP;
  extern __shared__ __align__(16) unsigned char ct_smem[];
  float (*xs)[68] = reinterpret_cast<float (*)[68]>(ct_smem);                   // [64][68] coordinate-major
  float (*ys)[YP] = reinterpret_cast<float (*)[YP]>(ct_smem + L::XS);           // [128][YP]
  float* xx = reinterpret_cast<float*>(ct_smem + L::XS + L::YS);               // [64]
  float* yyb = xx + 64;                                                         // [2][128]
  __shared__ double red[4];
  const int item = blockIdx.x;
  const int c = item_cl[item];
  const int tid = threadIdx.x;
  const int ti = tid & 7, tj = tid >> 3;
  const int64_t p_beg = off[item_mb[item]], p_end = off[item_mb[item + 1]];
  const int dpad = (d + 3) & ~3;
  const int pieces = dpad >> 2;
  auto load_chunk = [&](int64_t q0) {
    const int np = (int)((p_end - q0) < 128 ? (p_end - q0) : 128);
    for (int v = tid; v < np * pieces; v += 128) {
      const int j = v / pieces, k = v - j * pieces;
      cp_async16(&ys[j][4 * k], Y + (q0 + j) * dy + 4 * k);
    }
    cp_async_commit();
  };
  double acc = 0.0;
  for (int rb = 0; rb < ld; rb += 64) {
    __syncthreads();
    if (p_beg < p_end) load_chunk(p_beg);
    for (int v = tid; v < 64 * 64; v += 128) {
      const int t = v >> 6, i = v & 63;
      xs[t][i] = (rb + i < m && t < d) ? x[((int64_t)c * m + rb + i) * d + t] : 0.f;
    }
    __syncthreads();
    if (tid < 64) {
      float s = 0.f;
      for (int t = 0; t < d; ++t) s = fmaf(xs[t][tid], xs[t][tid], s);
      xx[tid] = s;
    }
    int buf = 0;
    for (int64_t q0 = p_beg; q0 < p_end; q0 += 128, buf ^= 1) {
      const int np = (int)((p_end - q0) < 128 ? (p_end - q0) : 128);
      cp_async_wait<0>();
      __syncthreads();
      float* yy = yyb + 128 * buf;
      {                                                // |y_j|^2 of point tid: 16-byte row reads, t in order
        float s = 0.f;
        for (int t = 0; t < dpad; t += 4) {
          const float4 v = *reinterpret_cast<const float4*>(&ys[tid][t]);
          if (t < d) s = fmaf(v.x, v.x, s);
          if (t + 1 < d) s = fmaf(v.y, v.y, s);
          if (t + 2 < d) s = fmaf(v.z, v.z, s);
          if (t + 3 < d) s = fmaf(v.w, v.w, s);
        }
        yy[tid] = s;
      }
      float2 a2[4][8];                                 // row pairs (4ti,+1) (4ti+2,+3) (32+4ti,+1) (32+4ti+2,+3) x 8 points
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) a2[u][v] = make_float2(0.f, 0.f);
      for (int t = 0; t < dpad; t += 4) {
        float4 y4[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) y4[v] = *reinterpret_cast<const float4*>(&ys[(v < 4 ? 4 * tj + v : 60 + 4 * tj + v)][t]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 xa = *reinterpret_cast<const float4*>(&xs[t + k][4 * ti]);
          const float4 xb = *reinterpret_cast<const float4*>(&xs[t + k][32 + 4 * ti]);
          const float2 x0 = make_float2(xa.x, xa.y), x1 = make_float2(xa.z, xa.w);
          const float2 x2 = make_float2(xb.x, xb.y), x3 = make_float2(xb.z, xb.w);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const float yk = k == 0 ? y4[v].x : (k == 1 ? y4[v].y : (k == 2 ? y4[v].z : y4[v].w));
            const float2 y2 = make_float2(yk, yk);
            a2[0][v] = __ffma2_rn(x0, y2, a2[0][v]);
            a2[1][v] = __ffma2_rn(x1, y2, a2[1][v]);
            a2[2][v] = __ffma2_rn(x2, y2, a2[2][v]);
            a2[3][v] = __ffma2_rn(x3, y2, a2[3][v]);
          }
        }
      }
      __syncthreads();                                 // yy ready; every read of ys[buf] done
      if (q0 + 128 < p_end) load_chunk(q0 + 128);     // the next chunk lands during the epilogue
      float s = 0.f;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int j = v < 4 ? 4 * tj + v : 60 + 4 * tj + v;
#pragma unroll
        for (int h = 0; h < 2; ++h) {                  // row halves 4ti.. and 32 + 4ti..
          const int r0 = rb + 32 * h + 4 * ti;
          if (j < np && r0 < ld) {
            float4 o;
            float* oe = reinterpret_cast<float*>(&o);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int i = r0 + u;
              const float2 pr = a2[2 * h + (u >> 1)][v];
              const float dot = (u & 1) ? pr.y : pr.x;
              const float cv = (i < m) ? fmaxf(fmaf(-2.f, dot, xx[i - rb] + yy[j]), 0.f) : 0.f;
              oe[u] = cv;
              s += cv;
            }
            *reinterpret_cast<float4*>(Cc + (q0 + j) * ld + r0) = o;
          }
        }
      }
      acc += (double)s;
    }
  }
  if (psum) {
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < 4; ++w) t += red[w];
      psum[item] = t;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// d > 64 (the paper's document embeddings, d = 300-400) for the cached-cost kernels
// ---------------------------------------------------------------------------------------------
// Cost build C_ij = |x_i|^2 + |y_j|^2 - 2 x_i.y_j with the coordinates in chunks of 64:
// per chunk of 64 points, X_c^T and the points' coordinates are staged 64 dims at a time and the
// 4 x 4 register tiles accumulate across the dim chunks; |x|^2, |y|^2 in fp32.  Rows >= m are 0,
// rows >= ld not written; per-item double sums for rho.  One CTA (256 threads) per work item.
__global__ void __launch_bounds__(256)
k_cost_tile_big(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
                const int32_t* __restrict__ item_cl, const float* __restrict__ Y, const float* __restrict__ x,
                float* __restrict__ Cc, double* __restrict__ psum, int m, int d, int dy, int ld) {
  __shared__ __align__(16) float xs[64][68];
  __shared__ __align__(16) float ys[64][68];
  __shared__ float xx[64], yy[64];
  __shared__ double red[8];
  const int item = blockIdx.x;
  const int c = item_cl[item];
  const int tid = threadIdx.x;
  const int ti = tid & 15, tj = tid >> 4;
  const int64_t p_beg = off[item_mb[item]], p_end = off[item_mb[item + 1]];
  double acc = 0.0;
  for (int rb = 0; rb < ld; rb += 64) {                // row blocks of 64 (ld = 128 for m > 64)
  __syncthreads();
  if (tid < 64) {
    float s = 0.f;
    if (rb + tid < m)
      for (int t = 0; t < d; ++t) {
        const float v = x[((int64_t)c * m + rb + tid) * d + t];
        s = fmaf(v, v, s);
      }
    xx[tid] = s;
  }
  for (int64_t q0 = p_beg; q0 < p_end; q0 += 64) {
    const int np = (int)((p_end - q0) < 64 ? (p_end - q0) : 64);
    float2 a2[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) a2[u][v] = make_float2(0.f, 0.f);
    float ysq = 0.f;                                   // |y|^2 of point tid (tid < 64)
    for (int t0 = 0; t0 < d; t0 += 64) {
      __syncthreads();                                 // previous chunk consumed
      for (int v = tid; v < 64 * 64; v += 256) {
        const int t = v >> 6, i = v & 63;
        xs[t][i] = (rb + i < m && t0 + t < d) ? x[((int64_t)c * m + rb + i) * d + t0 + t] : 0.f;
        const int j = v >> 6, tt = v & 63;
        ys[tt][j] = (j < np && t0 + tt < d) ? Y[(q0 + j) * dy + t0 + tt] : 0.f;
      }
      __syncthreads();
      if (tid < 64)
        for (int t = 0; t < 64; ++t) ysq = fmaf(ys[t][tid], ys[t][tid], ysq);
#pragma unroll 4
      for (int t = 0; t < 64; ++t) {
        const float4 xv = *reinterpret_cast<const float4*>(&xs[t][4 * ti]);
        const float4 yv = *reinterpret_cast<const float4*>(&ys[t][4 * tj]);
        const float2 x01 = make_float2(xv.x, xv.y), x23 = make_float2(xv.z, xv.w);
        const float ya[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float2 y2 = make_float2(ya[v], ya[v]);
          a2[0][v] = __ffma2_rn(x01, y2, a2[0][v]);
          a2[1][v] = __ffma2_rn(x23, y2, a2[1][v]);
        }
      }
    }
    if (tid < 64) yy[tid] = ysq;
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = 4 * tj + v;
      if (j < np && rb + 4 * ti < ld) {
        float o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = rb + 4 * ti + u;
          const float dot = (u & 1) ? a2[u >> 1][v].y : a2[u >> 1][v].x;
          o[u] = (i < m) ? fmaxf(fmaf(-2.f, dot, xx[i - rb] + yy[j]), 0.f) : 0.f;
          s += o[u];
        }
        *reinterpret_cast<float4*>(Cc + (q0 + j) * ld + rb + 4 * ti) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    acc += (double)s;
  }
  }
  if (psum) {
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      psum[item] = t;
    }
  }
}

// Support-update partials for d > 64 (Eq.updatex, X5): px[item*parts][i][t] = sum over the
// item's points j of Pi2_ij y_jt, px[..][i][d] = sum_j Pi2_ij, from the Pi2 blocks (Q,
// column-major, ld rows, contiguous over the item's points) and the supports.  Tiles of 64 rows x
// 64 coordinates, points in chunks of 32 staged in shared memory, 4 x 4 register tiles; the
// item's other part rows are zeroed (k_xsum adds all parts).  One CTA (256 threads) per item.
__global__ void __launch_bounds__(256)
k_xpart(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb, const float* __restrict__ Q,
        const float* __restrict__ Y, float* __restrict__ px, int m, int d, int dy, int ld, int parts) {
  __shared__ __align__(16) float qs[32][68];           // [point][row]
  __shared__ __align__(16) float ys[32][68];           // [point][coordinate]
  const int item = blockIdx.x;
  const int tid = threadIdx.x;
  const int ti = tid & 15, tj = tid >> 4;               // rows 4ti.., coordinates 4tj..
  const int64_t p_beg = off[item_mb[item]], p_end = off[item_mb[item + 1]];
  float* out = px + (int64_t)item * parts * m * (d + 1);
  for (int e = tid + m * (d + 1); e < parts * m * (d + 1); e += 256) out[e] = 0.f;   // parts 1..
  for (int rb = 0; rb < ld; rb += 64)                    // row blocks of 64 (ld = 128 for m > 64)
  for (int t0 = 0; t0 < d + 1; t0 += 64) {              // the last chunk holds the mass column d
    float a[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) a[u][v] = 0.f;
    for (int64_t q0 = p_beg; q0 < p_end; q0 += 32) {
      const int np = (int)((p_end - q0) < 32 ? (p_end - q0) : 32);
      __syncthreads();
      for (int v = tid; v < 32 * 64; v += 256) {
        const int j = v >> 6, r = v & 63;
        qs[j][r] = (j < np && rb + r < m) ? Q[(q0 + j) * ld + rb + r] : 0.f;
        const int t = t0 + r;
        ys[j][r] = (j < np) ? (t < d ? Y[(q0 + j) * dy + t] : (t == d ? 1.f : 0.f)) : 0.f;
      }
      __syncthreads();
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const float4 qv = *reinterpret_cast<const float4*>(&qs[j][4 * ti]);
        const float4 yv = *reinterpret_cast<const float4*>(&ys[j][4 * tj]);
        const float qa[4] = {qv.x, qv.y, qv.z, qv.w}, ya[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a[u][v] = fmaf(qa[u], ya[v], a[u][v]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = rb + 4 * ti + u;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int t = t0 + 4 * tj + v;
        if (i < m && t <= d) out[(int64_t)i * (d + 1) + t] = a[u][v];
      }
    }
  }
}

}  // namespace ad2k
