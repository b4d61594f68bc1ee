// ad2_assign.cu — the assignment step of AD2-clustering on the GPU:
//
//   l^(k) = argmin_c W_2^2(P_c, P^(k))           (Alg. 1; ties to the lowest c, X13)
//
// W_2^2 is the exact optimal-transport cost (Eq.primal) with the squared Euclidean
// ground cost, between centroid c (m points, weights w_c) and member k (m_k points, weights
// w^(k)), both renormalised in fp64.  One warp per member, everything in fp64:
//   1. lower bound for every centroid from the means: W^2 >= |mean(P_c) - mean(P^(k))|^2
//      (the squared-Euclidean cost splits into the distance of the means plus a non-negative
//      term);
//   2. centroids are visited in increasing bound order until the bound exceeds the best exact
//      cost found (Elkan-style pruning, without the inter-centroid table); for each
//      visited centroid the cost matrix is built and the relaxed-marginal bounds
//      sum_j w_j min_i C_ij and sum_i w_i min_j C_ij (each drops one constraint of Eq.primal)
//      prune again;
//   3. survivors are solved exactly by successive shortest paths on the bipartite transport
//      network (Dijkstra with node potentials on reduced costs, augment along the path by the
//      bottleneck of supply, demand and reverse-arc flow) — a primal-dual method that ends at
//      an optimal basic plan, so the cost equals the oracle's transportation simplex up to fp64
//      rounding.
// No float atomics: per-member results are written by the member's warp.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "../../include/ad2.h"

namespace ad2a {

// row stride of the fp32 cost copy used by the Sinkhorn sweeps: a multiple of 4 floats with an odd
// number of 16-byte groups, so lane-per-row LDS.128 reads are conflict-free (and lane-per-column
// scalar reads are consecutive)
__host__ __device__ inline int ldf_of(int mk) {
  int l = (mk + 3) & ~3;
  if (((l >> 2) & 1) == 0) l += 4;
  return l;
}

struct AsgLay {
  int m, mk, V, K, d;
  size_t oC, oF, opi, odist, oprev, odone, oarem, obrem, oom, oLB, osolv, oyb, oCf, olog, olb, oAb, oBb, oys, bytes;
  __host__ __device__ void make(int m_, int mk_, int K_, int d_) {
    m = m_, mk = mk_, K = K_, d = d_;
    V = m + mk;
    size_t o = 0;
    auto take = [&](size_t b) {
      size_t r = o;
      o += (b + 15) & ~(size_t)15;
      return r;
    };
    oC = take(8 * (size_t)m * (mk | 1));       // rows padded to an odd stride (bank-conflict-free columns)
    size_t fb = 8 * (size_t)m * (mk | 1);                 // flows; also the fp32 cost copy and
    if (4 * (size_t)m * ldf_of(mk) > fb) fb = 4 * (size_t)m * ldf_of(mk);   // the staged member
    if (8 * (size_t)mk * d > fb) fb = 8 * (size_t)mk * d;                    // points (aliases)
    oF = take(fb);
    opi = take(8 * (size_t)V);
    odist = take(8 * (size_t)V);
    oprev = take(4 * (size_t)V);
    odone = take(4 * (size_t)V);
    oarem = take(8 * (size_t)m);
    obrem = take(8 * (size_t)mk);
    oom = take(8 * (size_t)mk);
    oLB = take(8 * (size_t)K);
    osolv = take(4 * (size_t)((K + 31) / 32));
    oyb = take(8 * (size_t)d);
    oCf = oF;                                         // fp32 copy of C (Sinkhorn only) aliases the flows
    olog = take(4 * (size_t)m);                       // Sinkhorn: log a [m]
    olb = take(4 * (size_t)(mk + 4));                  // log b [m_k] (+ padding)
    oAb = take(4 * (size_t)m);                         // per-iteration row terms (base 2)
    oBb = take(4 * (size_t)(mk + 4));                  // per-iteration column terms (base 2)
    oys = oF;                                         // the member's points in fp64, staged per build_cost
    bytes = o;
  }
};

__device__ __forceinline__ float ex2f(float a) {      // MUFU 2^a (flush-to-zero)
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// order-preserving map of fp64 onto uint64 (negative values flip every bit, others the sign bit)
__device__ __forceinline__ unsigned long long okey(double x) {
  const long long b = __double_as_longlong(x);
  return (unsigned long long)(b ^ ((b >> 63) | (long long)0x8000000000000000ull));
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k ^ 0x8000000000000000ull) : ~k));
}

// exact W^2 by successive shortest paths; C row-major m x mk in smem; returns the cost of the
// final plan.  err bit 1: no augmenting path / iteration cap (should not happen on a balanced
// problem).
// warm: start from the dual-feasible potentials (u, v) that dual_bounds(duals_only) left in the
// pi region (pi_i = -u_i, pi_{m+j} = v_j, so every forward reduced cost C_ij - u_i - v_j >= 0);
// with near-optimal duals each Dijkstra reaches a sink over (near-)tight arcs in a few steps.
// The optimum does not depend on the starting potentials, only their feasibility.
__device__ __noinline__ double ssp_w2(const AsgLay& L, unsigned char* ws, const double* wn, int mk, int lane, int* err,
                         bool warm, unsigned long long* stats) {
  unsigned naug = 0, nstep = 0;
  const int m = L.m, V = m + mk, ld = mk | 1;
  const double* C = reinterpret_cast<const double*>(ws + L.oC);
  double* F = reinterpret_cast<double*>(ws + L.oF);
  double* pi = reinterpret_cast<double*>(ws + L.opi);
  double* dist = reinterpret_cast<double*>(ws + L.odist);
  int* prev = reinterpret_cast<int*>(ws + L.oprev);
  int* done = reinterpret_cast<int*>(ws + L.odone);
  double* arem = reinterpret_cast<double*>(ws + L.oarem);
  double* brem = reinterpret_cast<double*>(ws + L.obrem);
  const double* om = reinterpret_cast<const double*>(ws + L.oom);
  const double tiny = 1e-14;
  for (int e = lane; e < m * ld; e += 32) F[e] = 0.0;
  if (warm) {
    for (int i = lane; i < m; i += 32) pi[i] = -pi[i];
  } else {
    for (int v = lane; v < V; v += 32) pi[v] = 0.0;
  }
  for (int i = lane; i < m; i += 32) arem[i] = wn[i];
  for (int j = lane; j < mk; j += 32) brem[j] = om[j];
  __syncwarp();
  const int cap = 8 * V + 256;
  for (int it = 0;; ++it) {
    bool hs = false, hd = false;
    for (int i = lane; i < m; i += 32) hs |= arem[i] > tiny;
    for (int j = lane; j < mk; j += 32) hd |= brem[j] > tiny;
    if (!__any_sync(0xffffffffu, hs) || !__any_sync(0xffffffffu, hd)) break;
    if (it >= cap) {
      if (lane == 0) atomicOr(err, 1);
      break;
    }
    // every source with supply left is at distance 0: settle them all at once and relax their
    // forward arcs in one pass (lane = sink), instead of one Dijkstra step per source
    for (int i = lane; i < m; i += 32) {
      const bool act = arem[i] > tiny;
      done[i] = act;
      prev[i] = -1;
      dist[i] = act ? 0.0 : CUDART_INF;
    }
    for (int j = lane; j < mk; j += 32) {
      double bd = CUDART_INF;
      int bi = -1;
      const double pj = pi[m + j];
#pragma unroll 1
      for (int i = 0; i < m; ++i)
        if (arem[i] > tiny) {
          const double nd = C[i * ld + j] + pi[i] - pj;
          if (nd < bd) {
            bd = nd;
            bi = i;
          }
        }
      done[m + j] = 0;
      prev[m + j] = bi;
      dist[m + j] = bd;
    }
    __syncwarp();
    int t = -1;
    double dt = CUDART_INF;
    for (int step = 0; step < V; ++step) {
      // warp argmin of dist over unsettled nodes: order-preserving 64-bit keys, one shuffle
      // pair per round; the lowest lane holding the minimum key supplies the node (deterministic)
      unsigned long long key = ~0ull;
      int bv = V;
      for (int v = lane; v < V; v += 32)
        if (!done[v]) {
          const unsigned long long kv = okey(dist[v]);
          if (kv < key) {
            key = kv;
            bv = v;
          }
        }
      unsigned long long km = key;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long ok = __shfl_xor_sync(0xffffffffu, km, o);
        km = ok < km ? ok : km;
      }
      if (km == ~0ull) break;
      const int src = __ffs(__ballot_sync(0xffffffffu, key == km)) - 1;
      bv = __shfl_sync(0xffffffffu, bv, src);
      const double bd = okey_inv(km);
      if (bv >= V || !(bd < CUDART_INF)) break;
      if (lane == 0) done[bv] = 1;
      ++nstep;
      if (bv >= m && brem[bv - m] > tiny) {         // the nearest sink with demand left
        t = bv;
        dt = bd;
        __syncwarp();
        break;
      }
      __syncwarp();
      if (bv >= m) {                                // sink j: reverse arcs j -> i carrying flow
        const int j = bv - m;
        for (int i = lane; i < m; i += 32)
          if (!done[i] && F[i * ld + j] > 0.0) {
            const double nd = bd - C[i * ld + j] + pi[bv] - pi[i];
            if (nd < dist[i]) {
              dist[i] = nd;
              prev[i] = bv;
            }
          }
      } else {                                      // source i: forward arcs i -> j
        const int i = bv;
        for (int j = lane; j < mk; j += 32) {
          const int v = m + j;
          if (!done[v]) {
            const double nd = bd + C[i * ld + j] + pi[i] - pi[v];
            if (nd < dist[v]) {
              dist[v] = nd;
              prev[v] = i;
            }
          }
        }
      }
      __syncwarp();
    }
    if (t < 0) {
      if (lane == 0) atomicOr(err, 1);
      break;
    }
    ++naug;
    for (int v = lane; v < V; v += 32) pi[v] += done[v] ? dist[v] : dt;   // reduced costs stay >= 0
    __syncwarp();
    if (lane == 0) {
      double del = brem[t - m];
      int v = t;
      while (prev[v] >= 0) {
        const int u = prev[v];
        if (u >= m) del = fmin(del, F[v * ld + (u - m)]);
        v = u;
      }
      const int s = v;
      del = fmin(del, arem[s]);
      v = t;
      while (prev[v] >= 0) {
        const int u = prev[v];
        if (u < m) F[u * ld + (v - m)] += del;
        else F[v * ld + (u - m)] -= del;
        v = u;
      }
      arem[s] -= del;
      brem[t - m] -= del;
    }
    __syncwarp();
  }
  if (lane == 0) {                                  // statistics: augmentations, Dijkstra steps
    atomicAdd(stats, (unsigned long long)naug);
    atomicAdd(stats + 1, (unsigned long long)nstep);
  }
  double acc = 0.0;
#pragma unroll 1
  for (int i = 0; i < m; ++i)
    for (int j = lane; j < mk; j += 32) acc += F[i * ld + j] * C[i * ld + j];
  return wsum(acc);
}

// The same successive-shortest-path solve with the Dijkstra state in registers: lane l owns
// sources l + 32q and sinks l + 32q (q < Q, so m, m_k <= 32 Q); distances, settled flags and the
// own potentials live in registers, the node argmin is a 64-bit order-preserving key reduced by
// two 32-bit warp reductions (high word, then low word among the lanes holding the minimum high
// word) and the lowest such lane supplies the node.  Only prev (for the path walk), pi (broadcast
// of the settled node's potential) and the plan F stay in shared memory.  Warm start, bulk settle
// of the sources with supply and the augmentation step are those of ssp_w2.
template <int Q>
__device__ __noinline__ double ssp_reg(const AsgLay& L, unsigned char* ws, const double* wn, int mk, int lane,
                                       int* err, unsigned long long* stats) {
  const int m = L.m, V = m + mk, ld = mk | 1;
  const double* C = reinterpret_cast<const double*>(ws + L.oC);
  double* F = reinterpret_cast<double*>(ws + L.oF);
  double* pi = reinterpret_cast<double*>(ws + L.opi);
  int* prev = reinterpret_cast<int*>(ws + L.oprev);
  double* arem = reinterpret_cast<double*>(ws + L.oarem);
  double* brem = reinterpret_cast<double*>(ws + L.obrem);
  const double* om = reinterpret_cast<const double*>(ws + L.oom);
  const double tiny = 1e-14;
  unsigned naug = 0, nstep = 0;
  for (int e = lane; e < m * ld; e += 32) F[e] = 0.0;
  for (int i = lane; i < m; i += 32) {
    pi[i] = -pi[i];                                  // warm start: pi_i = -u_i, pi_{m+j} = v_j
    arem[i] = wn[i];
  }
  for (int j = lane; j < mk; j += 32) brem[j] = om[j];
  __syncwarp();
  double ps[Q], pk[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int i = lane + 32 * q, j = lane + 32 * q;
    ps[q] = i < m ? pi[i] : 0.0;
    pk[q] = j < mk ? pi[m + j] : 0.0;
  }
  const int cap = 8 * V + 256;
  for (int it = 0;; ++it) {
    bool hs = false, hd = false;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = lane + 32 * q;
      hs |= i < m && arem[i] > tiny;
      hd |= i < mk && brem[i] > tiny;
    }
    if (!__any_sync(0xffffffffu, hs) || !__any_sync(0xffffffffu, hd)) break;
    if (it >= cap) {
      if (lane == 0) atomicOr(err, 1);
      break;
    }
    double ds[Q], dk[Q];
    unsigned dn = 0;                                 // settled: bit q source, bit Q + q sink
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = lane + 32 * q;
      const bool act = i < m && arem[i] > tiny;
      ds[q] = act ? 0.0 : CUDART_INF;
      if (act || i >= m) dn |= 1u << q;
      if (i < m) prev[i] = -1;
    }
    // the sources with supply left, compacted in index order (ballot prefix counts)
    int* act = reinterpret_cast<int*>(ws + L.odone);
    int nact = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int i = lane + 32 * q;
      const bool a_ = i < m && arem[i] > tiny;
      const unsigned bal = __ballot_sync(0xffffffffu, a_);
      if (a_) act[nact + __popc(bal & ((1u << lane) - 1u))] = i;
      nact += __popc(bal);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int j = lane + 32 * q;
      double bd = CUDART_INF;
      int bi = -1;
      if (j < mk) {
        // four independent running minima (sources t = r mod 4), merged lowest index first
        double b4[4] = {CUDART_INF, CUDART_INF, CUDART_INF, CUDART_INF};
        int i4[4] = {-1, -1, -1, -1};
        int t = 0;
#pragma unroll 1
        for (; t + 4 <= nact; t += 4) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int i = act[t + r];
            const double nd = C[i * ld + j] + pi[i] - pk[q];
            if (nd < b4[r]) {
              b4[r] = nd;
              i4[r] = i;
            }
          }
        }
#pragma unroll 1
        for (; t < nact; ++t) {
          const int i = act[t];
          const double nd = C[i * ld + j] + pi[i] - pk[q];
          if (nd < b4[0]) {
            b4[0] = nd;
            i4[0] = i;
          }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (b4[r] < bd || (b4[r] == bd && i4[r] >= 0 && i4[r] < bi)) {
            bd = b4[r];
            bi = i4[r];
          }
        prev[m + j] = bi;
      } else {
        dn |= 1u << (Q + q);
      }
      dk[q] = bd;
    }
    int t = -1;
    double dt = CUDART_INF;
    for (int step = 0; step < V; ++step) {
      unsigned long long key = ~0ull;
      int cand = V;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if (!((dn >> q) & 1u)) {
          const unsigned long long kv = okey(ds[q]);
          if (kv < key) {
            key = kv;
            cand = lane + 32 * q;
          }
        }
        if (!((dn >> (Q + q)) & 1u)) {
          const unsigned long long kv = okey(dk[q]);
          if (kv < key) {
            key = kv;
            cand = m + lane + 32 * q;
          }
        }
      }
      const unsigned hi = (unsigned)(key >> 32);
      const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
      const unsigned lo = hi == mh ? (unsigned)key : 0xffffffffu;
      const unsigned ml = __reduce_min_sync(0xffffffffu, lo);
      if (mh == 0xffffffffu && ml == 0xffffffffu) break;
      const unsigned ball = __ballot_sync(0xffffffffu, hi == mh && lo == ml);
      const int bv = __shfl_sync(0xffffffffu, cand, __ffs(ball) - 1);
      const double bd = okey_inv(((unsigned long long)mh << 32) | ml);
      if (bv >= V || !(bd < CUDART_INF)) break;
      ++nstep;
      const bool snk = bv >= m;
      const int nid = snk ? bv - m : bv;
      if ((nid & 31) == lane) dn |= 1u << ((snk ? Q : 0) + (nid >> 5));
      if (snk && brem[nid] > tiny) {                 // the nearest sink with demand left
        t = bv;
        dt = bd;
        break;
      }
      const double pb = pi[bv];
      if (snk) {                                     // reverse arcs j -> i carrying flow
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int i = lane + 32 * q;
          if (!((dn >> q) & 1u) && F[i * ld + nid] > 0.0) {
            const double nd = bd - C[i * ld + nid] + pb - ps[q];
            if (nd < ds[q]) {
              ds[q] = nd;
              prev[i] = bv;
            }
          }
        }
      } else {                                       // forward arcs i -> j
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int j = lane + 32 * q;
          if (!((dn >> (Q + q)) & 1u)) {
            const double nd = bd + C[nid * ld + j] + pb - pk[q];
            if (nd < dk[q]) {
              dk[q] = nd;
              prev[m + j] = nid;
            }
          }
        }
      }
    }
    if (t < 0) {
      if (lane == 0) atomicOr(err, 1);
      break;
    }
    ++naug;
#pragma unroll
    for (int q = 0; q < Q; ++q) {                   // reduced costs stay >= 0
      const int i = lane + 32 * q;
      if (i < m) {
        ps[q] += ((dn >> q) & 1u) ? ds[q] : dt;
        pi[i] = ps[q];
      }
      if (i < mk) {
        pk[q] += ((dn >> (Q + q)) & 1u) ? dk[q] : dt;
        pi[m + i] = pk[q];
      }
    }
    __syncwarp();
    if (lane == 0) {
      double del = brem[t - m];
      int v = t;
      while (prev[v] >= 0) {
        const int u = prev[v];
        if (u >= m) del = fmin(del, F[v * ld + (u - m)]);
        v = u;
      }
      const int s0 = v;
      del = fmin(del, arem[s0]);
      v = t;
      while (prev[v] >= 0) {
        const int u = prev[v];
        if (u < m) F[u * ld + (v - m)] += del;
        else F[v * ld + (u - m)] -= del;
        v = u;
      }
      arem[s0] -= del;
      brem[t - m] -= del;
    }
    __syncwarp();
  }
  if (lane == 0) {
    atomicAdd(stats, (unsigned long long)naug);
    atomicAdd(stats + 1, (unsigned long long)nstep);
  }
  double acc = 0.0;
#pragma unroll 1
  for (int i = 0; i < m; ++i)
    for (int j = lane; j < mk; j += 32) acc += F[i * ld + j] * C[i * ld + j];
  return wsum(acc);
}

// Dual lower bound and primal upper bound on W^2 for one pair (C in smem, fp64).  A log-domain
// Sinkhorn run (fp32, eps-scaling from max C down to 1e-3 mean C) gives
// approximate potentials f (24 iterations); two c-transforms in fp64 make them dual-feasible
// (v_j = min_i C_ij - u_i, u_i = min_j C_ij - v_j, so u_i + v_j <= C_ij), hence
// LB = sum_i a_i u_i + sum_j b_j v_j <= W^2 (Kantorovich duality).  The Sinkhorn plan rounded
// onto the transport polytope (row scaling to <= a, column scaling to <= b, rank-one
// correction, Altschuler et al.) is feasible, hence UB = <C, P> >= W^2.  Uses F as scratch.
// dual-feasible potentials from fs by two fp64 c-transforms -> Kantorovich lower bound
__device__ __noinline__ double ctrans_lb(int m, int mk, const double* C, const float* fs, const double* a, const double* b,
                            double* u, double* v, int lane) {
  const int ld = mk | 1;
  for (int j = lane; j < mk; j += 32) {
    double mn = CUDART_INF;
#pragma unroll 1
    for (int i = 0; i < m; ++i) mn = fmin(mn, C[i * ld + j] - (double)fs[i]);
    v[j] = mn;
  }
  __syncwarp();
  double acc = 0.0;
  for (int i = lane; i < m; i += 32) {
    double mn = CUDART_INF;
#pragma unroll 1
    for (int j = 0; j < mk; ++j) mn = fmin(mn, C[i * ld + j] - v[j]);
    u[i] = mn;
    acc += a[i] * mn;
  }
  for (int j = lane; j < mk; j += 32) acc += b[j] * v[j];
  const double r = wsum(acc);
  __syncwarp();
  return r;
}

// Kantorovich lower bound from zero potentials by two fp64 c-transforms, in both orders
// (v_j = min_i C_ij, u_i = min_j C_ij - v_j; and the mirror), each dual-feasible — at least the
// relaxed-marginal bounds sum_j b_j min_i C_ij and sum_i a_i min_j C_ij, for O(m m_k) work.
__device__ __noinline__ double zero_ctrans_lb(int m, int mk, const double* C, const double* a, const double* b, double* u,
                                 double* v, int lane) {
  const int ld = mk | 1;
  for (int j = lane; j < mk; j += 32) {
    double mn = CUDART_INF;
#pragma unroll 1
    for (int i = 0; i < m; ++i) mn = fmin(mn, C[i * ld + j]);
    v[j] = mn;
  }
  for (int i = lane; i < m; i += 32) {
    double mn = CUDART_INF;
#pragma unroll 1
    for (int j = 0; j < mk; ++j) mn = fmin(mn, C[i * ld + j]);
    u[i] = mn;
  }
  __syncwarp();
  double a1 = 0.0, a2 = 0.0;
  for (int i = lane; i < m; i += 32) {
    double mn = CUDART_INF;
#pragma unroll 1
    for (int j = 0; j < mk; ++j) mn = fmin(mn, C[i * ld + j] - v[j]);
    a1 += a[i] * mn;
    a2 += a[i] * u[i];
  }
  for (int j = lane; j < mk; j += 32) {
    double mn = CUDART_INF;
#pragma unroll 1
    for (int i = 0; i < m; ++i) mn = fmin(mn, C[i * ld + j] - u[i]);
    a1 += b[j] * v[j];
    a2 += b[j] * mn;
  }
  const double r = fmax(wsum(a1), wsum(a2));
  __syncwarp();
  return r;
}

// prune_at: if an intermediate lower bound (after 8 / 16 iterations) already exceeds it, return
// early with ub = +inf (the candidate cannot win)
// duals_only: stop after the lower bound, leaving the dual-feasible (u, v) in the pi region
__device__ __noinline__ void dual_bounds(const AsgLay& L, unsigned char* ws, const double* a, int mk, int lane, double prune_at,
                            double& lb, double& ub, bool duals_only = false, unsigned long long* iters = nullptr) {
  const int m = L.m, ld = mk | 1;
  const double* C = reinterpret_cast<const double*>(ws + L.oC);
  double* P = reinterpret_cast<double*>(ws + L.oF);
  double* u = reinterpret_cast<double*>(ws + L.opi);          // [m] then v at u + m
  double* v = u + m;
  float* fs = reinterpret_cast<float*>(ws + L.odist);         // f [m], g [mk] (fp32 potentials)
  float* gs = fs + m;
  float* Cf = reinterpret_cast<float*>(ws + L.oCf);            // fp32 copy of C, row stride ldf
  float* la = reinterpret_cast<float*>(ws + L.olog);           // log a [m]
  float* lbv = reinterpret_cast<float*>(ws + L.olb);           // log b [m_k]
  float* Ab = reinterpret_cast<float*>(ws + L.oAb);            // (log a_i + f_i / eps) log2 e
  float* Bb = reinterpret_cast<float*>(ws + L.oBb);            // (log b_j + g_j / eps) log2 e; -inf pad
  const double* b = reinterpret_cast<const double*>(ws + L.oom);
  const int ldf = ldf_of(mk), nq = (mk + 3) >> 2;
  double cmax = 0.0, csum = 0.0;
#pragma unroll 1
  for (int i = 0; i < m; ++i)
    for (int j = lane; j < ldf; j += 32) {
      float cf = 0.f;
      if (j < mk) {
        const double c = C[i * ld + j];
        cmax = fmax(cmax, c);
        csum += c;
        cf = (float)c;
      }
      Cf[i * ldf + j] = cf;
    }
  for (int i = lane; i < m; i += 32) la[i] = __logf((float)a[i] + 1e-38f);
  for (int j = lane; j < mk; j += 32) lbv[j] = __logf((float)b[j] + 1e-38f);
  for (int j = mk + lane; j < 4 * nq; j += 32) Bb[j] = -CUDART_INF_F;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
  csum = wsum(csum);
  const float eps_f = (float)fmax(1e-3 * csum / (double)(m * mk), 1e-30);
  float eps = (float)fmax(0.25 * cmax, 1e-30);          // first iteration at cmax / 8
  for (int i = lane; i < m; i += 32) fs[i] = 0.f;
  for (int j = lane; j < mk; j += 32) gs[j] = 0.f;
  __syncwarp();
  const float L2E = 1.4426950408889634f, LN2 = 0.6931471805599453f;
  for (int it = 0; it < 24; ++it) {
    eps = fmaxf(eps_f, eps * 0.5f);
    const float ie = 1.f / eps, iel = ie * L2E;
    // g_j = -eps LSE_i(log a_i + (f_i - C_ij)/eps), in base 2: t_ij = Ab_i - C_ij iel
    for (int i = lane; i < m; i += 32) Ab[i] = (la[i] + fs[i] * ie) * L2E;
    __syncwarp();
    for (int j = lane; j < mk; j += 32) {
      float mx = -CUDART_INF_F;
      for (int i = 0; i < m; ++i) mx = fmaxf(mx, fmaf(-Cf[i * ldf + j], iel, Ab[i]));
      float sm = 0.f;
      for (int i = 0; i < m; ++i) sm += ex2f(fmaf(-Cf[i * ldf + j], iel, Ab[i]) - mx);
      gs[j] = -eps * LN2 * (mx + __log2f(sm));
    }
    __syncwarp();
    // f_i = -eps LSE_j(log b_j + (g_j - C_ij)/eps): lane = row, four columns per LDS.128
    for (int j = lane; j < mk; j += 32) Bb[j] = (lbv[j] + gs[j] * ie) * L2E;
    __syncwarp();
    for (int i = lane; i < m; i += 32) {
      const float4* cr = reinterpret_cast<const float4*>(Cf + i * ldf);
      const float4* br = reinterpret_cast<const float4*>(Bb);
      float mx = -CUDART_INF_F;
      for (int q = 0; q < nq; ++q) {
        const float4 c4 = cr[q], b4 = br[q];
        mx = fmaxf(mx, fmaxf(fmaxf(fmaf(-c4.x, iel, b4.x), fmaf(-c4.y, iel, b4.y)),
                             fmaxf(fmaf(-c4.z, iel, b4.z), fmaf(-c4.w, iel, b4.w))));
      }
      float s0 = 0.f, s1 = 0.f;
      for (int q = 0; q < nq; ++q) {
        const float4 c4 = cr[q], b4 = br[q];
        s0 += ex2f(fmaf(-c4.x, iel, b4.x) - mx) + ex2f(fmaf(-c4.y, iel, b4.y) - mx);
        s1 += ex2f(fmaf(-c4.z, iel, b4.z) - mx) + ex2f(fmaf(-c4.w, iel, b4.w) - mx);
      }
      fs[i] = -eps * LN2 * (mx + __log2f(s0 + s1));
    }
    __syncwarp();
    if (it == 1 || it == 3 || it == 7 || it == 15) {   // early exit for clearly worse centroids
      const double l = ctrans_lb(m, mk, C, fs, a, b, u, v, lane);
      if (l * (1.0 - 1e-12) > prune_at) {
        lb = l;
        ub = CUDART_INF;
        if (iters && lane == 0) atomicAdd(iters, (unsigned long long)(it + 1));
        return;
      }
    }
  }
  lb = ctrans_lb(m, mk, C, fs, a, b, u, v, lane);
  if (iters && lane == 0) atomicAdd(iters, 24ull);
  if (duals_only) {
    ub = CUDART_INF;
    return;
  }
  // primal: Sinkhorn plan, rounded onto the transport polytope
  const float ie = 1.f / eps;
#pragma unroll 1
  for (int i = 0; i < m; ++i)
    for (int j = lane; j < mk; j += 32)
      P[i * ld + j] = (double)__expf((fs[i] + gs[j] - (float)C[i * ld + j]) * ie) * a[i] * b[j];
  __syncwarp();
  for (int i = lane; i < m; i += 32) {              // rows scaled down to <= a_i
    double r = 0.0;
#pragma unroll 1
    for (int j = 0; j < mk; ++j) r += P[i * ld + j];
    const double x = r > a[i] ? a[i] / r : 1.0;
#pragma unroll 1
    for (int j = 0; j < mk; ++j) P[i * ld + j] *= x;
  }
  __syncwarp();
  for (int j = lane; j < mk; j += 32) {             // columns scaled down to <= b_j
    double c = 0.0;
#pragma unroll 1
    for (int i = 0; i < m; ++i) c += P[i * ld + j];
    const double y = c > b[j] ? b[j] / c : 1.0;
#pragma unroll 1
    for (int i = 0; i < m; ++i) P[i * ld + j] *= y;
    v[j] = b[j] - c * y;                            // column deficit
  }
  __syncwarp();
  double dr = 0.0;
  for (int i = lane; i < m; i += 32) {
    double r = 0.0;
#pragma unroll 1
    for (int j = 0; j < mk; ++j) r += P[i * ld + j];
    u[i] = fmax(a[i] - r, 0.0);                     // row deficit
    dr += u[i];
  }
  dr = wsum(dr);
  __syncwarp();
  double cu = 0.0;
  const double idr = dr > 0.0 ? 1.0 / dr : 0.0;
#pragma unroll 1
  for (int i = 0; i < m; ++i)
    for (int j = lane; j < mk; j += 32) {
      const int e = i * ld + j;
      const double pe = P[e] + u[i] * fmax(v[j], 0.0) * idr;
      cu += C[e] * pe;
    }
  ub = wsum(cu);
}

// C_ij = |x_ci - y_j|^2 in fp64 (difference form) with lane = centroid row: x_i is held in
// registers 16 coordinates at a time, the member's points ys are broadcast from shared memory;
// symbolic supports read the table instead.
template <typename T>
__device__ __noinline__ void build_cost(const AsgLay& L, unsigned char* ws, const double* __restrict__ xk, int mk, int lane,
                           const int32_t* xs_c, const int32_t* Ysym, const double* Dtab, int V, int* err,
                           const T* __restrict__ Yk) {
  const int m = L.m, d = L.d, ld = mk | 1;
  double* C = reinterpret_cast<double*>(ws + L.oC);
  double* ys = reinterpret_cast<double*>(ws + L.oys);
  if (Dtab) {
#pragma unroll 1
    for (int i = 0; i < m; ++i)
      for (int j = lane; j < mk; j += 32) {
        const int e = i * ld + j;
        const int sa = xs_c[i], sb = Ysym[j];
        double a = 0.0;
        if (sa < 0 || sa >= V || sb < 0 || sb >= V) atomicOr(err, 4);
        else a = Dtab[(int64_t)sa * V + sb];
        C[e] = a;
      }
    return;
  }
  for (int e = lane; e < mk * d; e += 32) ys[e] = (double)Yk[e];   // ys shares the flows' region
  __syncwarp();
  for (int i = lane; i < m; i += 32) {
    for (int t0 = 0; t0 < d; t0 += 16) {
      double xr[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) xr[t] = (t0 + t < d) ? xk[(int64_t)i * d + t0 + t] : 0.0;
      const int tn = d - t0 < 16 ? d - t0 : 16;
#pragma unroll 1
      for (int j = 0; j < mk; ++j) {
        const double* yj = ys + j * d + t0;
        double a = (t0 == 0) ? 0.0 : C[i * ld + j];
#pragma unroll
        for (int t = 0; t < 16; ++t)
          if (t < tn) {
            const double df = xr[t] - yj[t];
            a += df * df;
          }
        C[i * ld + j] = a;
      }
    }
  }
}

// centroids to fp64: weights renormalised by their (sequential) fp64 sum, weighted means
// (x == nullptr: symbolic supports, weights only)
template <typename T>
__global__ void k_assign_prep(const T* __restrict__ x, const T* __restrict__ w, int K, int m, int d,
                              double* __restrict__ xc, double* __restrict__ wc, double* __restrict__ xb) {
  const int c = blockIdx.x;
  __shared__ double tot;
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll 1
    for (int i = 0; i < m; ++i) s += (double)w[(int64_t)c * m + i];
    tot = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) wc[(int64_t)c * m + i] = (double)w[(int64_t)c * m + i] / tot;
  if (!x) return;
  for (int e = threadIdx.x; e < m * d; e += blockDim.x) xc[(int64_t)c * m * d + e] = (double)x[(int64_t)c * m * d + e];
  __syncthreads();
  for (int t = threadIdx.x; t < d; t += blockDim.x) {
    double s = 0.0;
#pragma unroll 1
    for (int i = 0; i < m; ++i) s += wc[(int64_t)c * m + i] * xc[((int64_t)c * m + i) * d + t];
    xb[(int64_t)c * d + t] = s;
  }
}

// validation + largest m_k (err bit 2: offsets[0] != 0 or m_k < 1)
__global__ void k_assign_mk(const int64_t* __restrict__ off, int64_t N, unsigned long long* mkmax, int* err) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0 && off[0] != 0) atomicOr(err, 2);
  if (k >= N) return;
  const int64_t mk = off[k + 1] - off[k];
  if (mk < 1 || mk > 0x7fffffff) atomicOr(err, 2);
  else atomicMax(mkmax, (unsigned long long)mk);
}

// Dtab != nullptr: symbolic supports — Y and xs hold int32 symbol ids, the cost is the
// table entry D[xs_ci][y_j] (fp64 copy), and there is no vector-space mean bound (all bounds 0:
// centroids are visited in index order, the relaxed-marginal bounds still prune).
// Cross-round pruning (Elkan; AsgBounds) with W = sqrt(W^2), a metric: skip[k]
// certifies member k's label (lab_in[k]) and the member is not visited; otherwise the search
// starts from the carried lower bounds lb[k][c] <= W(P_k, Q_c) (prior != 0) and writes back
// u[k] >= W(P_k, Q_label) and lb[k][c] for every centroid (W units, rounded down in fp32).
// fixed != nullptr: only the exact W^2 to centroid fixed[k] (label = fixed[k]).
struct AsgBounds {
  const uint8_t* skip;
  const int32_t* lab_in;
  const int32_t* fixed;
  double* u;
  float* lb;
  int prior;
};

template <typename T>
__global__ void k_assign(const int64_t* __restrict__ off, int64_t N, const T* __restrict__ Y,
                         const T* __restrict__ Wt, const double* __restrict__ xc, const double* __restrict__ wc,
                         const double* __restrict__ xb, const int32_t* __restrict__ xs, const double* __restrict__ Dtab,
                         int V, AsgLay L, int32_t* __restrict__ labels,
                         double* __restrict__ best_out, unsigned long long* __restrict__ n_exact, int* err,
                         AsgBounds bnd) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ws = smem + (size_t)warp * L.bytes;
  // persistent warps: members are taken from a global counter (n_exact[5]) one at a time, so
  // a warp with cheap members moves on instead of idling until its block's slowest warp ends
  for (;;) {
    unsigned long long kq = 0;
    if (lane == 0) kq = atomicAdd(n_exact + 5, 1ull);
    const int64_t k = (int64_t)__shfl_sync(0xffffffffu, kq, 0);
    if (k >= N) break;
    if (bnd.skip && bnd.skip[k]) {                    // certified: the label holds, nothing to solve
      if (lane == 0) labels[k] = bnd.lab_in[k];
      continue;
    }
    const int m = L.m, K = L.K, d = L.d;
    double* C = reinterpret_cast<double*>(ws + L.oC);
    double* om = reinterpret_cast<double*>(ws + L.oom);
    double* LB = reinterpret_cast<double*>(ws + L.oLB);
    unsigned* solved = reinterpret_cast<unsigned*>(ws + L.osolv);
    double* yb = reinterpret_cast<double*>(ws + L.oyb);
    const int64_t o0 = off[k];
    const int mk = (int)(off[k + 1] - o0), ld = mk | 1;
    const T* Yk = Y + o0 * d;

    // member weights renormalised in fp64 (O1), member mean
    double s = 0.0;
    for (int j = lane; j < mk; j += 32) s += (double)Wt[o0 + j];
    s = wsum(s);
    for (int j = lane; j < mk; j += 32) om[j] = (double)Wt[o0 + j] / s;
    __syncwarp();
    const int32_t* Ysym = reinterpret_cast<const int32_t*>(Y) + o0;
    if (!Dtab)
      for (int t = lane; t < d; t += 32) {
        double a = 0.0;
#pragma unroll 1
        for (int j = 0; j < mk; ++j) a += om[j] * (double)Yk[(int64_t)j * d + t];
        yb[t] = a;
      }
    if (bnd.fixed) {                                   // one exact W^2 (e.g. a centroid's drift)
      const int cs = bnd.fixed[k];
      const double* wn = wc + (int64_t)cs * m;
      build_cost(L, ws, xc + (int64_t)cs * m * d, mk, lane, Dtab ? xs + (int64_t)cs * m : nullptr, Ysym, Dtab, V, err, Yk);
      __syncwarp();
      double dlb, dub;
      dual_bounds(L, ws, wn, mk, lane, CUDART_INF, dlb, dub, true);
      const int qn = ((m > mk ? m : mk) + 31) >> 5;
      const double W = qn <= 1   ? ssp_reg<1>(L, ws, wn, mk, lane, err, n_exact + 3)
                       : qn <= 2 ? ssp_reg<2>(L, ws, wn, mk, lane, err, n_exact + 3)
                       : qn <= 4 ? ssp_reg<4>(L, ws, wn, mk, lane, err, n_exact + 3)
                                 : ssp_w2(L, ws, wn, mk, lane, err, true, n_exact + 3);
      if (lane == 0) {
        labels[k] = cs;
        if (best_out) best_out[k] = W;
        atomicAdd(n_exact, 1ull);
      }
      __syncwarp();
      continue;
    }
    for (int q = lane; q < (K + 31) / 32; q += 32) solved[q] = 0u;
    __syncwarp();
    for (int c = lane; c < K; c += 32) {              // |mean_c - mean_k|^2 <= W^2
      double a = 0.0;
      if (!Dtab)
        for (int t = 0; t < d; ++t) {
          const double df = xb[(int64_t)c * d + t] - yb[t];
          a += df * df;
        }
      if (bnd.lb && bnd.prior) {                      // the carried Elkan bound, W^2 units
        const double e = fmax((double)bnd.lb[k * K + c], 0.0);
        a = fmax(a, e * e * (1.0 - 1e-12));
      }
      LB[c] = a;
    }
    __syncwarp();
    const double shrink = 1.0 - 1e-12;               // fp64 rounding margin on the bounds
    const double grow = 1.0 + 1e-9;                  // margin on the rounded-plan upper bound
    double best = CUDART_INF;
    int bc = -1;
    unsigned nsolve = 0, nvisit = 0;
    // phase A: candidates in increasing mean-bound order while the mean bound is below the best
    // upper bound: sharpen each bound (relaxed marginals, Sinkhorn dual) and collect upper bounds
    double ubest = CUDART_INF;
    for (int visit = 0; visit < K; ++visit) {
      __syncwarp();
      double lb = CUDART_INF;
      int cs = K;
      for (int c = lane; c < K; c += 32)
        if (!((solved[c >> 5] >> (c & 31)) & 1u) && LB[c] < lb) {
          lb = LB[c];
          cs = c;
        }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const double ol = __shfl_xor_sync(0xffffffffu, lb, o);
        const int oc = __shfl_xor_sync(0xffffffffu, cs, o);
        if (ol < lb || (ol == lb && oc < cs)) {
          lb = ol;
          cs = oc;
        }
      }
      if (cs >= K || lb * shrink > ubest) break;      // every remaining centroid has W^2 > ubest
      build_cost(L, ws, xc + (int64_t)cs * m * d, mk, lane, Dtab ? xs + (int64_t)cs * m : nullptr, Ysym, Dtab, V, err, Yk);
      __syncwarp();
      const double* wn = wc + (int64_t)cs * m;
      double dlb, dub;
      const double zlb = zero_ctrans_lb(m, mk, C, wn, om, reinterpret_cast<double*>(ws + L.opi),
                                        reinterpret_cast<double*>(ws + L.opi) + m, lane);
      if (zlb * shrink > ubest) {                      // cannot win: no Sinkhorn run
        dlb = zlb;
        dub = CUDART_INF;
      } else {
        dual_bounds(L, ws, wn, mk, lane, ubest, dlb, dub, false, n_exact + 6);   // [7]: Sinkhorn iterations
        dlb = fmax(dlb, zlb);
        ++nvisit;
      }
      ubest = fmin(ubest, dub * grow);
      if (lane == 0) {
        LB[cs] = fmax(lb, dlb);                       // sharpened bound (cs stays unsolved)
        solved[cs >> 5] |= 1u << (cs & 31);           // visited in phase A
      }
      __syncwarp();
    }
    // phase B: only phase-A centroids can win (the others have mean bound > ubest >= the best
    // exact W^2, so the loop below stops before reaching them; their mean bounds stay in LB as
    // lower bounds for the pruning of the next round); exact solves in increasing sharpened-bound
    // order until the bound exceeds the best exact W^2
    for (int q = lane; q < (K + 31) / 32; q += 32) solved[q] = 0u;
    __syncwarp();
    for (int visit = 0; visit < K; ++visit) {
      __syncwarp();                                   // C / solved of the previous visit consumed
      double lb = CUDART_INF;
      int cs = K;
      for (int c = lane; c < K; c += 32)
        if (!((solved[c >> 5] >> (c & 31)) & 1u) && LB[c] < lb) {
          lb = LB[c];
          cs = c;
        }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const double ol = __shfl_xor_sync(0xffffffffu, lb, o);
        const int oc = __shfl_xor_sync(0xffffffffu, cs, o);
        if (ol < lb || (ol == lb && oc < cs)) {
          lb = ol;
          cs = oc;
        }
      }
      if (cs >= K) break;
      const double lbs = lb * shrink;
      if (lbs > best || (lbs == best && cs > bc)) break;            // no remaining centroid can win
      if (lane == 0) solved[cs >> 5] |= 1u << (cs & 31);
      // cost matrix C_ij = |x_ci - y_j|^2, difference form in fp64
      build_cost(L, ws, xc + (int64_t)cs * m * d, mk, lane, Dtab ? xs + (int64_t)cs * m : nullptr, Ysym, Dtab, V, err, Yk);
      __syncwarp();
      // relaxed-marginal lower bounds
      const double* wn = wc + (int64_t)cs * m;
      double l1 = 0.0, l2 = 0.0;
      for (int j = lane; j < mk; j += 32) {
        double mn = CUDART_INF;
#pragma unroll 1
        for (int i = 0; i < m; ++i) mn = fmin(mn, C[i * ld + j]);
        l1 += om[j] * mn;
      }
      for (int i = lane; i < m; i += 32) {
        double mn = CUDART_INF;
#pragma unroll 1
        for (int j = 0; j < mk; ++j) mn = fmin(mn, C[i * ld + j]);
        l2 += wn[i] * mn;
      }
      const double lbr = fmax(wsum(l1), wsum(l2)) * shrink;
      if (lane == 0) LB[cs] = fmax(LB[cs], lbr);
      if (lbr > best || (lbr == best && cs > bc)) continue;
      double dlb, dub;
      dual_bounds(L, ws, wn, mk, lane, CUDART_INF, dlb, dub, true);
      const int qn = ((m > mk ? m : mk) + 31) >> 5;
      const double W = qn <= 1   ? ssp_reg<1>(L, ws, wn, mk, lane, err, n_exact + 3)
                       : qn <= 2 ? ssp_reg<2>(L, ws, wn, mk, lane, err, n_exact + 3)
                       : qn <= 4 ? ssp_reg<4>(L, ws, wn, mk, lane, err, n_exact + 3)
                                 : ssp_w2(L, ws, wn, mk, lane, err, true, n_exact + 3);
      ++nsolve;
      if (lane == 0) LB[cs] = W;                        // exact
      if (W < best || (W == best && cs < bc)) {
        best = W;
        bc = cs;
      }
      __syncwarp();
    }
    if (bnd.u) {
      // Elkan bounds in W units with rounding margins: u >= W(P_k, Q_bc) (exact here); lb[k][c] <=
      // W(P_k, Q_c): exact where solved, else the sharpened / mean / carried lower bound
      __syncwarp();
      for (int c = lane; c < K; c += 32)
        bnd.lb[k * K + c] = __double2float_rd(sqrt(fmax(LB[c], 0.0)) * (1.0 - 1e-9));
      if (lane == 0) bnd.u[k] = sqrt(fmax(best, 0.0)) * (1.0 + 1e-9) + 1e-300;
    }
    if (lane == 0) {
      labels[k] = bc;
      if (best_out) best_out[k] = best;
      atomicAdd(n_exact, (unsigned long long)nsolve);
      atomicAdd(n_exact + 2, (unsigned long long)nvisit);   // scal[3]: phase-A candidates (statistics)
    }
    __syncwarp();
  }
}

}  // namespace ad2a

using namespace ad2a;

size_t assign_warp_bytes(int m, int mkmax, int K, int d) {
  AsgLay L;
  L.make(m, mkmax, K, d);
  return L.bytes;
}

// x, w: device centroids in the batch dtype; all pointers device
template <typename T>
__global__ void k_to_f64(const T* __restrict__ a, double* __restrict__ b, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = (double)a[i];
}

// symbolic (xs != nullptr): x unused, Y / xs int32 ids, table D [V][V] in the batch dtype
int assign_launch(int f64, const int64_t* off, int64_t N, const void* Y, const void* Wt, const void* x,
                  const void* w, int K, int m, int d, int mkmax, double* xc, double* wc, double* xb,
                  const int32_t* xs, const void* D, int V, double* Dtab,
                  int32_t* labels, double* best, unsigned long long* n_exact, int* err, int optin, cudaStream_t s,
                  const uint8_t* skip, const int32_t* lab_in, const int32_t* fixed, double* bu, float* blb,
                  int prior) {
  const AsgBounds bnd{skip, lab_in, fixed, bu, blb, prior};
  if (f64) k_assign_prep<double><<<K, 128, 0, s>>>(xs ? nullptr : (const double*)x, (const double*)w, K, m, d, xc, wc, xb);
  else k_assign_prep<float><<<K, 128, 0, s>>>(xs ? nullptr : (const float*)x, (const float*)w, K, m, d, xc, wc, xb);
  if (xs) {
    const int64_t nv = (int64_t)V * V;
    if (f64) k_to_f64<double><<<(unsigned)((nv + 255) / 256), 256, 0, s>>>((const double*)D, Dtab, nv);
    else k_to_f64<float><<<(unsigned)((nv + 255) / 256), 256, 0, s>>>((const float*)D, Dtab, nv);
  }
  if (N == 0) return 0;
  AsgLay L;
  L.make(m, mkmax, K, d);
  // one warp per block (independent workspaces), as many resident blocks as shared memory allows
  // (at most 16 per SM: the register limit), a persistent grid of SMs x blocks per SM
  if (L.bytes + 1024 > (size_t)optin) return -1;
  int dev = 0, nsm = 0, smem_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  int bps = (int)((size_t)smem_sm / (L.bytes + 1024));
  bps = bps < 1 ? 1 : (bps > 16 ? 16 : bps);
  const int wpc = 1;
  const size_t sm = L.bytes;
  int64_t nb = (int64_t)nsm * bps;
  if (nb > N) nb = N;
  const unsigned grid = (unsigned)nb;
  if (f64) {
    cudaFuncSetAttribute(k_assign<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_assign<double><<<grid, 32 * wpc, sm, s>>>(off, N, (const double*)Y, (const double*)Wt, xc, wc, xb, xs,
                                                xs ? Dtab : nullptr, V, L, labels, best, n_exact, err, bnd);
  } else {
    cudaFuncSetAttribute(k_assign<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_assign<float><<<grid, 32 * wpc, sm, s>>>(off, N, (const float*)Y, (const float*)Wt, xc, wc, xb, xs,
                                               xs ? Dtab : nullptr, V, L, labels, best, n_exact, err, bnd);
  }
  return 0;
}

// ---- cross-round pruning (Elkan) -------------------------------------------------
// drift2[c] = W^2(Q_c^old, Q_c^new) (exact).  One warp per member: lb[k][c] -= delta_c (rounded
// down), u[k] += delta_label; certified when every other centroid's lower bound exceeds u.
__global__ void k_elkan_update(const int32_t* __restrict__ lab, int64_t N, int K, const double* __restrict__ drift2,
                               double* __restrict__ u, float* __restrict__ lb, uint8_t* __restrict__ skip,
                               unsigned long long* __restrict__ n_skip) {
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (k >= N) return;
  const int lk = lab[k];
  auto delta = [&](int c) { return sqrt(fmax(drift2[c], 0.0)) * (1.0 + 1e-9) + 1e-300; };
  const double uu = (u[k] + delta(lk)) * (1.0 + 1e-15);
  float mn = CUDART_INF_F;
  for (int c = lane; c < K; c += 32) {
    const float v = __double2float_rd((double)lb[k * K + c] - delta(c));
    lb[k * K + c] = v;
    if (c != lk) mn = fminf(mn, v);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) {
    u[k] = uu;
    const bool ok = (double)mn > uu;
    skip[k] = ok ? 1 : 0;
    if (ok) atomicAdd(n_skip, 1ull);
  }
}

void elkan_launch(const double* drift2, int K, const int32_t* lab, int64_t N, double* u, float* lb, uint8_t* skip,
                  unsigned long long* n_skip, cudaStream_t s) {
  if (N > 0) k_elkan_update<<<(unsigned)((N + 7) / 8), 256, 0, s>>>(lab, N, K, drift2, u, lb, skip, n_skip);
}

void assign_mkmax(const int64_t* off, int64_t N, unsigned long long* mkmax, int* err, cudaStream_t s) {
  if (N == 0) return;
  k_assign_mk<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(off, N, mkmax, err);
}

// ------------------------------------------------------------------------------------------
// Centroid initialisation by Eq.merge: one warp per cluster c takes the chosen
// member pick[c] (renormalised weights, fp64) and merges the pair (i < j) minimising
// w_i w_j |x_i - x_j|^2 / (w_i + w_j) (lowest (i, j) on ties) into the weighted mean at i (j
// removed, later points move up) until m remain; with fewer than m points the heaviest point
// (lowest index on ties) is split into two halves, the copy appended (reading X19).
// ------------------------------------------------------------------------------------------
namespace ad2a {
__global__ void k_pick_sizes(const int64_t* __restrict__ off, const int64_t* __restrict__ pick, int K, int64_t N,
                             int64_t* __restrict__ mk, int* __restrict__ err) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K) return;
  const int64_t k = pick[c];
  if (k < 0 || k >= N) {
    atomicOr(err, 8);
    mk[c] = 0;
    return;
  }
  mk[c] = off[k + 1] - off[k];
}

template <typename T>
__global__ void k_merge_init(const int64_t* __restrict__ off, const T* __restrict__ Y, const T* __restrict__ Wt,
                             const int64_t* __restrict__ pick, int m, int d, int cap, T* __restrict__ x0,
                             T* __restrict__ w0) {
  extern __shared__ __align__(16) double msm[];
  double* x = msm;                                  // [cap][d]
  double* w = msm + (size_t)cap * d;                // [cap]
  const int c = blockIdx.x, lane = threadIdx.x;
  const int64_t k = pick[c];
  const int64_t o0 = off[k];
  const int mk = (int)(off[k + 1] - o0);
  double s = 0.0;
  if (lane == 0)
    for (int j = 0; j < mk; ++j) s += (double)Wt[o0 + j];
  s = __shfl_sync(0xffffffffu, s, 0);
  for (int j = lane; j < mk; j += 32) w[j] = (double)Wt[o0 + j] / s;
  for (int e = lane; e < mk * d; e += 32) x[e] = (double)Y[o0 * d + e];
  __syncwarp();
  int n = mk;
  while (n > m) {
    double best = CUDART_INF;
    int bp = 1 << 30;
    const int np = n * (n - 1) / 2;
    for (int p = lane; p < np; p += 32) {           // pair p -> (i, j), i < j, in (i, j) order
      int i = 0, rem = p;
      while (rem >= n - 1 - i) {
        rem -= n - 1 - i;
        ++i;
      }
      const int j = i + 1 + rem;
      // uncontracted IEEE operations in the oracle's order: identical decisions
      double dd = 0.0;
      for (int t = 0; t < d; ++t) {
        const double df = __dsub_rn(x[i * d + t], x[j * d + t]);
        dd = __dadd_rn(dd, __dmul_rn(df, df));
      }
      const double cst = __ddiv_rn(__dmul_rn(__dmul_rn(w[i], w[j]), dd), __dadd_rn(w[i], w[j]));
      if (cst < best) {                             // pairs of a lane ascend: first minimum kept
        best = cst;
        bp = p;
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (ob < best || (ob == best && op < bp)) {
        best = ob;
        bp = op;
      }
    }
    int bi = 0, rem = bp;
    while (rem >= n - 1 - bi) {
      rem -= n - 1 - bi;
      ++bi;
    }
    const int bj = bi + 1 + rem;
    const double wb = w[bi] + w[bj];
    __syncwarp();
    for (int t = lane; t < d; t += 32)
      x[bi * d + t] = __ddiv_rn(__dadd_rn(__dmul_rn(w[bi], x[bi * d + t]), __dmul_rn(w[bj], x[bj * d + t])), wb);
    __syncwarp();
    if (lane == 0) {
      w[bi] = wb;
      for (int j = bj; j < n - 1; ++j) {
        w[j] = w[j + 1];
        for (int t = 0; t < d; ++t) x[j * d + t] = x[(j + 1) * d + t];
      }
    }
    --n;
    __syncwarp();
  }
  if (lane == 0) {
    while (n < m) {
      int h = 0;
      for (int j = 1; j < n; ++j)
        if (w[j] > w[h]) h = j;
      w[h] *= 0.5;
      w[n] = w[h];
      for (int t = 0; t < d; ++t) x[n * d + t] = x[h * d + t];
      ++n;
    }
    double tot = 0.0;
    for (int i = 0; i < m; ++i) tot += w[i];
    for (int i = 0; i < m; ++i) w[i] = w[i] / tot;
  }
  __syncwarp();
  for (int i = lane; i < m; i += 32) w0[(int64_t)c * m + i] = (T)w[i];
  for (int e = lane; e < m * d; e += 32) x0[(int64_t)c * m * d + e] = (T)x[e];
}
}  // namespace ad2a

int merge_init_launch(int f64, const int64_t* off, const void* Y, const void* Wt, const int64_t* pick, int K, int m,
                      int d, int cap, void* x0, void* w0, int optin, cudaStream_t s) {
  const size_t sm = sizeof(double) * ((size_t)cap * d + cap);
  if (sm > (size_t)optin) return -1;
  if (f64) {
    cudaFuncSetAttribute(k_merge_init<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_merge_init<double><<<K, 32, sm, s>>>(off, (const double*)Y, (const double*)Wt, pick, m, d, cap, (double*)x0,
                                          (double*)w0);
  } else {
    cudaFuncSetAttribute(k_merge_init<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_merge_init<float><<<K, 32, sm, s>>>(off, (const float*)Y, (const float*)Wt, pick, m, d, cap, (float*)x0,
                                         (float*)w0);
  }
  return 0;
}

void pick_sizes_launch(const int64_t* off, const int64_t* pick, int K, int64_t N, int64_t* mk, int* err, cudaStream_t s) {
  k_pick_sizes<<<(K + 127) / 128, 128, 0, s>>>(off, pick, K, N, mk, err);
}
