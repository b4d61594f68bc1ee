// ad2_kernels.cuh — sm_100a kernels of the modified B-ADMM barycenter path (arXiv 1510.00012,
// Alg. 4).  "P:n" = PAPER.md line n.  Included only by ad2.cu.
//
// Device layout: members are sorted by cluster; member s owns
// the contiguous column-major m x m_s block [m*off[s], m*off[s+1]) of every plan-shaped array
// (Pi^(1) in P, Pi^(2) in Q, Lambda in L, cost C in Cc): entry (i, j) at m*off[s] + j*m + i.
// This is the paper's Pi in R^{m x n} with column j = member support point j.
//
// Iteration kernels run per work item = a run of consecutive members of ONE cluster; each item
// writes its own partial sums (no float atomics), and the cluster reduction kernels add the
// items of a cluster in item order, so every result is deterministic.
#pragma once
#include <cuda_runtime.h>
#include <cstdio>
#include <type_traits>
#include <math_constants.h>
#include <stdint.h>

namespace ad2k {

// P1INIT: P1ONLY at the start of a cold round (variant-2 kernel): Pi2^0 = w_i w_j^(k)
// and Lambda = 0 are formed in registers instead of being written by k_init_plans and read back
// P2X: P2ONLY without the stores (the support-update partials only); the next step starts with a
// FUSED pass that recomputes the same phase 2 (variant-2 kernel)
// FUSEDX: FUSED that also forms the support-update partials of the Pi2 its phase 1 implies
// (x_i = mean over members of sum_j (pe_ij + eps) y_j / r_i, w_i cancels): the last pass of a step
// Epoch-anchored compressed state, variant 2, steps of >= 3:
// with the eps of Eq.badmmc0b/c1b dropped from the Pi2 recursion, Lambda cancels between them
// and Pi2^t = G (.) exp(-s C / rho) (.) a_i b_j from an anchor G = Pi2^{t0}
// (pin P4).  Between launches the state is G (read-only), U = Lambda + rho Pi1 (one array) and
// per-member log-factors ra [N][ld], cb [n]:
// GIN: FUSED that stores G = Pi2^{t-1} (exact, with eps) into Q and U, ra, cb instead of Pi1, Lambda
// GMID: Pi2^{t-1} from (G, ra, cb), then phase 1; stores U, ra, cb (12 B/entry instead of 16)
// GXOUT: GMID's phase 2 and phase 1 storing Pi1 and Lambda (the exact state again) + x partials
enum { P1ONLY = 0, FUSED = 1, P2ONLY = 2, P1INIT = 3, P2X = 4, FUSEDX = 5, GIN = 6, GMID = 7, GXOUT = 8 };
enum { ERR_NONFINITE = 1, ERR_WEIGHTS = 2, ERR_EPSCOL = 16 };   // ERR_EPSCOL: a flag, not an error

constexpr int NWARP = 4;          // warps per CTA in the warp-per-member kernels
// resident CTAs per SM of the fp32 16-row single-chunk small-d variant-2 build (k_badmm_tma)
#ifndef AD2_TMA_MINB16
#define AD2_TMA_MINB16 4
#endif

// Checked build (python -m paper_1510_00012_b200.build --checked -> libad2_checked.so): device
// assertions on the shared-memory ring placement and pass geometry of the staged kernels, a
// stand-in for compute-sanitizer (closed on the GPU pool).  Compiled out otherwise.
#ifdef AD2_CHECKS
#define AD2_CHECK(c)                                                                             \
  do {                                                                                           \
    if (!(c)) {                                                                                  \
      printf("AD2_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, blockIdx.x, \
             threadIdx.x, #c);                                                                   \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define AD2_CHECK(c) \
  do {               \
  } while (0)
#endif

// Programmatic dependent launch (the step graph of variant 2): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its predecessor drains;
// pdl_wait() blocks until the predecessor has completed and its writes are visible (a no-op for a
// normal launch), pdl_trigger() lets the successor's CTAs be scheduled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
constexpr int ITEM_PASSES = 8;    // member passes per warp per work item
constexpr int CT_WORDS = 32 + 32 + 64 + 8;   // doubles per cluster of the 3 x TF32 cost build's centres

// exp(v) is evaluated as ex(v * kx): kx = log2(e)/rho with MUFU ex2.approx for fp32,
// kx = 1/rho with the IEEE double exp for fp64 (fp64 has no MUFU path).
template <typename T> struct Num;
template <> struct Num<float> {
  static __device__ __forceinline__ float ex(float a) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
  }
  static __device__ __forceinline__ float ld(const float* p) { return __ldcs(p); }
  static __device__ __forceinline__ void st(float* p, float v) { __stcs(p, v); }
  // fp32 normalisations: MUFU reciprocal based quotient (<= 2 ulp), far inside the fp32 parity bar;
  // the operands are row / column masses >= m_k eps or m eps, far from the denormal range
  static __device__ __forceinline__ float div(float a, float b) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
    return a * r;
  }
  // kx * rho for kx = log2(e)/rho: the scale of a pre-scaled Lambda's dual step
  static __device__ __forceinline__ float kappa() { return 1.4426950408889634f; }
  // logarithm in the base of ex (log2), per row / column only: the accurate library function
  static __device__ __forceinline__ float lg(float a) { return log2f(a); }
};
template <> struct Num<double> {
  static __device__ __forceinline__ double ex(double a) { return exp(a); }
  static __device__ __forceinline__ double lg(double a) { return log(a); }
  static __device__ __forceinline__ double ld(const double* p) { return __ldcs(p); }
  static __device__ __forceinline__ void st(double* p, double v) { __stcs(p, v); }
  static __device__ __forceinline__ double div(double a, double b) { return a / b; }
  static __device__ __forceinline__ double kappa() { return 1.0; }
};

template <typename T>
struct IterArgs {
  const int64_t* off;      // [N+1] sorted member point offsets
  const int64_t* item_mb;  // [n_items+1] first sorted member of each item
  const int32_t* item_cl;  // [n_items] cluster of each item
  const T* Y;              // [n][d] supports, sorted
  const T* om;             // [n] member weights w^(k)_j, renormalised
  T* P;                    // Pi^(1)
  T* Q;                    // Pi^(2)
  T* L;                    // Lambda
  const T* Cc;             // cost C
  const T* w;              // [K][m] consensus weights
  const T* x;              // [K][m][d] centroid support points
  const T* rho;            // [K]
  const T* kx;             // [K] exponent scale (see Num)
  T* pw;                   // [n_items][m]   partial sum over members of wt (R1) or sqrt(wt) (R2)
  T* px;                   // [n_items][m][d+1] partial sums of pi2_ij y_j and pi2_ij
  int* err;
  int m, d, rule;
  int ld;                  // leading dimension of a member block (rows; >= m)
  int dy;                  // row stride of Y (>= d, zero-padded)
  int xext;                // 1: the x partials come from k_xpart (d > 64), P2ONLY skips them
  T eps;
  T* ra;                   // compressed state: [N][ld] row log-factors (GIN / GMID / GXOUT)
  T* cb;                   // compressed state: [n] column log-factors
  int gs;                  // compressed state: iterations since the anchor of this launch's phase 2
  int pdl;                 // host: launch with programmatic stream serialization (the kernel pdl_wait()s)
  int tc;                  // host: variant 2 with 32-row single-member passes and 4 < d <= 16 takes the
                           // tensor-core cost instantiation (ad2_set_tc_cost)
  const int32_t* perm;     // [n_items] work item of each CTA (full items first, then each cluster's
                           // partial last item, largest first: small items fill the launch's tail)
};

// 16-byte vectors of the element type (shared-memory tiles, staged rows)
template <typename T> struct Vec16;
template <> struct Vec16<float> {
  using type = float4;
  static __device__ __forceinline__ float hsum(float4 v) { return ((v.x + v.y) + v.z) + v.w; }
};
template <> struct Vec16<double> {
  using type = double2;
  static __device__ __forceinline__ double hsum(double2 v) { return v.x + v.y; }
};

// ---------------------------------------------------------------------------------------------
// Generic iteration kernel: any m, m_k, d.  One thread per member (work item = 1 member), state
// in global memory, row masses in a per-member scratch [2m].  Same MODE semantics as above.
// ---------------------------------------------------------------------------------------------
template <typename T, int MODE>
__global__ void __launch_bounds__(128)
k_badmm_generic(const IterArgs<T> a, T* __restrict__ scr, int64_t n_items) {
  using N = Num<T>;
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  const int64_t k = a.item_mb[it];                 // one member per item
  const int c = a.item_cl[it];
  const int m = a.m, d = a.d;
  const int64_t o0 = a.off[k];
  const int mk = (int)(a.off[k + 1] - o0);
  const int64_t base = (int64_t)m * o0;
  const T kx = a.kx[c], rho = a.rho[c], eps = a.eps;
  const T* w = a.w + (int64_t)c * m;
  T* r = scr + it * 2 * m;
  T* r2 = r + m;
  bool bad = false;
  if (MODE != P1ONLY) {
    for (int i = 0; i < m; ++i) {
      T s = T(0);
      for (int j = 0; j < mk; ++j) {
        const int64_t e = base + (int64_t)j * m + i;
        s += a.P[e] * N::ex(a.L[e] * kx) + eps;
      }
      r[i] = s;
    }
    if (MODE == P2ONLY) {
      T* px = a.px + it * m * (d + 1);
      for (int v = 0; v < m * (d + 1); ++v) px[v] = T(0);
    }
    for (int j = 0; j < mk; ++j)
      for (int i = 0; i < m; ++i) {
        const int64_t e = base + (int64_t)j * m + i;
        const T p = a.P[e];
        const T b = p * N::ex(a.L[e] * kx) + eps;
        const T q = b * (w[i] / r[i]);
        const T ln = a.L[e] + rho * (p - q);
        a.L[e] = ln;
        if (MODE == P2ONLY) {
          a.Q[e] = q;
          T* px = a.px + it * m * (d + 1) + (int64_t)i * (d + 1);
          for (int t = 0; t < d; ++t) px[t] += q * a.Y[(o0 + j) * d + t];
          px[d] += q;
        } else {
          a.P[e] = q * N::ex(-(a.Cc[e] + ln) * kx) + eps;      // pt2 stored in P for now
        }
      }
    if (MODE == P2ONLY) return;
  } else {
    for (int j = 0; j < mk; ++j)
      for (int i = 0; i < m; ++i) {
        const int64_t e = base + (int64_t)j * m + i;
        a.P[e] = a.Q[e] * N::ex(-(a.Cc[e] + a.L[e]) * kx) + eps;
      }
  }
  for (int i = 0; i < m; ++i) r2[i] = T(0);
  for (int j = 0; j < mk; ++j) {
    T s = T(0);
    for (int i = 0; i < m; ++i) s += a.P[base + (int64_t)j * m + i];
    const T f = a.om[o0 + j] / s;
    for (int i = 0; i < m; ++i) {
      const int64_t e = base + (int64_t)j * m + i;
      const T p = a.P[e] * f;
      a.P[e] = p;
      r2[i] += p * N::ex(a.L[e] * kx) + eps;
    }
  }
  T R = T(0);
  for (int i = 0; i < m; ++i) R += r2[i];
  for (int i = 0; i < m; ++i) {
    const T wt = r2[i] / R;
    bad |= !isfinite(wt);
    a.pw[it * m + i] = (a.rule == 1) ? sqrt(wt) : wt;
  }
  if (bad) atomicOr(a.err, ERR_NONFINITE);
}

// ---------------------------------------------------------------------------------------------
// Cluster reductions (one CTA per cluster, items added in item order).
// ---------------------------------------------------------------------------------------------
// w consensus: S_i = sum over the cluster's items of pw; with `finalize` (single rank) also
//   R1 (Eq.badmmw):  w_i = S_i / sum_i S_i          R2 (Eq.badmmw2): w_i = S_i^2 / sum_i S_i^2
// sum over rows it0, it0 + st, it0 + 2 st, ... < ie of column i of a row-major [rows][w] array,
// four independent accumulators (loads in flight together), combined in a fixed order
template <typename T>
__device__ __forceinline__ T slice_sum(const T* __restrict__ a, int64_t it0, int64_t ie, int st, int w, int i) {
  T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
  int64_t it = it0;
  for (; it + 3 * (int64_t)st < ie; it += 4 * (int64_t)st) {
    s0 += a[it * w + i];
    s1 += a[(it + st) * w + i];
    s2 += a[(it + 2 * st) * w + i];
    s3 += a[(it + 3 * st) * w + i];
  }
  for (; it < ie; it += st) s0 += a[it * w + i];
  return (s0 + s1) + (s2 + s3);
}

template <typename T>
__global__ void k_wsum(const T* __restrict__ pw, const int64_t* __restrict__ cl_item, int parts, int m,
                       T* __restrict__ S, T* __restrict__ w, int rule, int finalize, int* err) {
  // rows in passes of R = min(m, blockDim); S = blockDim/R slices take items s, s+S, ... in order,
  // then slice partials are added in slice order: deterministic for a fixed launch shape.
  const int c = blockIdx.x;
  const int64_t ib = cl_item[c] * parts, ie = cl_item[c + 1] * parts;   // `parts` partial rows per item
  pdl_wait();                                          // the iteration kernel's partials
  pdl_trigger();                                       // the next iteration kernel may start its set-up
  extern __shared__ unsigned char smraw[];
  T* red = reinterpret_cast<T*>(smraw);               // [blockDim]
  T* sh = red + blockDim.x;                            // [m]
  const int R = m < (int)blockDim.x ? m : (int)blockDim.x;
  const int NS = (int)blockDim.x / R;
  const int r = threadIdx.x % R, sl = threadIdx.x / R;
  for (int i0 = 0; i0 < m; i0 += R) {
    const int i = i0 + r;
    T s = T(0);
    if (sl < NS && i < m) s = slice_sum(pw, ib + sl, ie, NS, m, i);
    red[threadIdx.x] = s;
    __syncthreads();
    if (sl == 0 && i < m) {
      T t0 = T(0), t1 = T(0);
      int u = 0;
      for (; u + 1 < NS; u += 2) {
        t0 += red[u * R + r];
        t1 += red[(u + 1) * R + r];
      }
      if (u < NS) t0 += red[u * R + r];
      const T t = t0 + t1;
      S[(int64_t)c * m + i] = t;
      sh[i] = (rule == 1) ? t * t : t;
    }
    __syncthreads();
  }
  if (!finalize) return;
  __shared__ T tot;
  if (threadIdx.x == 0) {
    T t = T(0);
    for (int i = 0; i < m; ++i) t += sh[i];
    tot = t;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const T v = sh[i] / tot;
    if (!isfinite(v)) atomicOr(err, ERR_NONFINITE);
    w[(int64_t)c * m + i] = v;
  }
}

template <typename T>
__global__ void k_wfinal(const T* __restrict__ S, T* __restrict__ w, int m, int rule, int* err) {
  const int c = blockIdx.x;
  extern __shared__ unsigned char smraw[];
  T* sh = reinterpret_cast<T*>(smraw);
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const T s = S[(int64_t)c * m + i];
    sh[i] = (rule == 1) ? s * s : s;
  }
  __syncthreads();
  __shared__ T tot;
  if (threadIdx.x == 0) {
    T t = T(0);
    for (int i = 0; i < m; ++i) t += sh[i];
    tot = t;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const T v = sh[i] / tot;
    if (!isfinite(v)) atomicOr(err, ERR_NONFINITE);
    w[(int64_t)c * m + i] = v;
  }
}

// x partial sums -> Sx[K][m][d+1]
// (as k_wsum: elements in passes of R = min(W, blockDim), S = blockDim / R slices of the partial
// rows, slice sums added in slice order: deterministic for a fixed launch shape)
template <typename T>
__global__ void k_xsum(const T* __restrict__ px, const int64_t* __restrict__ cl_item, int parts, int m, int d,
                       T* __restrict__ Sx) {
  extern __shared__ unsigned char smraw[];
  T* red = reinterpret_cast<T*>(smraw);               // [blockDim]
  const int c = blockIdx.x;
  const int64_t ib = cl_item[c] * parts, ie = cl_item[c + 1] * parts;
  const int W = m * (d + 1);
  const int R = W < (int)blockDim.x ? W : (int)blockDim.x;
  const int NS = (int)blockDim.x / R;
  const int r = threadIdx.x % R, sl = threadIdx.x / R;
  for (int v0 = 0; v0 < W; v0 += R) {
    const int v = v0 + r;
    T s = T(0);
    if (sl < NS && v < W) s = slice_sum(px, ib + sl, ie, NS, W, v);
    red[threadIdx.x] = s;
    __syncthreads();
    if (sl == 0 && v < W) {
      T t0 = T(0), t1 = T(0);
      int u = 0;
      for (; u + 1 < NS; u += 2) {
        t0 += red[u * R + r];
        t1 += red[(u + 1) * R + r];
      }
      if (u < NS) t0 += red[u * R + r];
      Sx[(int64_t)c * W + v] = t0 + t1;
    }
    __syncthreads();
  }
}

// Eq.updatex (X5, X12): x_i = sum pi2_ij y_j / sum pi2_ij unless w_i < 1e-12
template <typename T>
__global__ void k_xfinal(const T* __restrict__ Sx, const T* __restrict__ w, T* __restrict__ x, int m,
                         int d) {
  const int c = blockIdx.x;
  for (int v = threadIdx.x; v < m * d; v += blockDim.x) {
    const int i = v / d, t = v - i * d;
    if (w[(int64_t)c * m + i] < T(1e-12)) continue;
    const T* s = Sx + ((int64_t)c * m + i) * (d + 1);
    x[((int64_t)c * m + i) * d + t] = s[t] / s[d];
  }
}

// ---------------------------------------------------------------------------------------------
// Cost build C_ij = sum_t (x_it - y_jt)^2 (difference form), optional per-item double
// sums of C for rho (Eq.rho, X1).  CTA per item, warp per member, lane per entry.
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128)
k_cost(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
       const int32_t* __restrict__ item_cl, const T* __restrict__ Y, const T* __restrict__ x,
       T* __restrict__ Cc, double* __restrict__ psum, int m, int d, int ld, int dy) {
  const int item = blockIdx.x;
  const int c = item_cl[item];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* xc = x + (int64_t)c * m * d;
  double acc = 0.0;
  for (int64_t k = item_mb[item] + warp; k < item_mb[item + 1]; k += 4) {
    const int64_t o0 = off[k];
    const int mk = (int)(off[k + 1] - o0);
    const int64_t base = (int64_t)ld * o0;
    for (int e = lane; e < ld * mk; e += 32) {
      const int j = e / ld, i = e - j * ld;
      T s = T(0);
      if (i < m)
        for (int t = 0; t < d; ++t) {
          const T df = xc[i * d + t] - Y[(o0 + j) * dy + t];
          s += df * df;
        }
      Cc[base + e] = s;
      acc += (double)s;
    }
  }
  if (psum) {
    for (int h = 16; h >= 1; h >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, h);
    __shared__ double sh[4];
    if (lane == 0) sh[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) psum[item] = sh[0] + sh[1] + sh[2] + sh[3];
  }
}


// surrogate objective partials (X14): sum_k <C, Pi1> per item, in double
template <typename T>
__global__ void __launch_bounds__(128)
k_objective(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
            const T* __restrict__ Cc, const T* __restrict__ P, double* __restrict__ psum, int ld) {
  const int item = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int64_t k = item_mb[item] + warp; k < item_mb[item + 1]; k += 4) {
    const int64_t base = (int64_t)ld * off[k];
    const int64_t ne = (int64_t)ld * (off[k + 1] - off[k]);
    T s = T(0);
    for (int64_t e = lane; e < ne; e += 32) s += Cc[base + e] * P[base + e];
    acc += (double)s;
  }
  for (int h = 16; h >= 1; h >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, h);
  __shared__ double sh[4];
  if (lane == 0) sh[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) psum[item] = sh[0] + sh[1] + sh[2] + sh[3];
}

// per-cluster sum of per-item doubles (fixed order)
static __global__ void k_dsum_cl(const double* __restrict__ psum, const int64_t* __restrict__ cl_item,
                          double* __restrict__ S, int K) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K) return;
  double s = 0.0;
  for (int64_t it = cl_item[c]; it < cl_item[c + 1]; ++it) s += psum[it];
  S[c] = s;
}

// rho_c = rho0 * sumC_c / (m * npts_c) (Eq.rho with X1); kx per Num
template <typename T>
__global__ void k_rho(const double* __restrict__ sumC, const double* __restrict__ npts, int K, int m,
                      double rho0, T* __restrict__ rho, T* __restrict__ kx, double* __restrict__ rho_d) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= K) return;
  const double r = rho0 * sumC[c] / ((double)m * npts[c]);
  rho_d[c] = r;
  rho[c] = (T)r;
  kx[c] = (sizeof(T) == 4) ? (T)(1.4426950408889634 / r) : (T)(1.0 / r);
}

// ---------------------------------------------------------------------------------------------
// Layout kernels: gather the caller's members into the cluster-sorted layout (renormalising the
// member weights), initial plans, and the state read-back in caller order.
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(128)
k_gather(const int32_t* __restrict__ order, const int64_t* __restrict__ src_off,
         const int64_t* __restrict__ dst_off, const T* __restrict__ Ysrc, const T* __restrict__ Wsrc,
         T* __restrict__ Y, T* __restrict__ om, int64_t N, int d, int dy, int yy_col, double wtol, int* err,
         const double* __restrict__ xsum, const int32_t* __restrict__ mem_cl, int m, double* __restrict__ pm) {
  // warp per member, lane per support point: the point's row [y, 0.., |y|^2 at yy_col, 0..]
  const int64_t s = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= N) return;
  const int64_t k = order[s];
  const int64_t so = src_off[k], dsto = dst_off[s];
  const int mk = (int)(src_off[k + 1] - so);
  // coordinates: the member's source block is contiguous, read lane-strided (coalesced)
  const T* srcb = Ysrc + so * d;
  T* dstb = Y + dsto * dy;
  // (with pm: the Eq.rho numerator of the member in the same pass, fp64, closed form:
  //  sum_ij |x_i - y_j|^2 = m_k sum_i |x_i|^2 + sum_jt (m y_jt^2 - 2 (sum_i x_it) y_jt), the cluster's
  //  sums from k_xsums; fp32 inputs are exact in fp64)
  const double* xs = pm ? xsum + (int64_t)mem_cl[s] * (d + 1) : nullptr;
  double racc = 0.0;
  {
    // element e = lane + 32 q of the block: (j, t) advanced incrementally (no integer division)
    const int dj = 32 / d, dt = 32 % d;
    int j = lane / d, t = lane - (lane / d) * d;
    for (int e = lane; e < mk * d; e += 32) {
      const T v = srcb[e];
      dstb[(int64_t)j * dy + t] = v;
      if (pm) racc += (double)v * fma((double)m, (double)v, -2.0 * xs[t]);
      j += dj;
      t += dt;
      if (t >= d) {
        t -= d;
        ++j;
      }
    }
  }
  // zero padding and the |y|^2 column (sequential in t, like the oracle's sum): lane per point
  if (dy > d)
    for (int j = lane; j < mk; j += 32) {
      const T* src = srcb + (int64_t)j * d;
      T* dst = dstb + (int64_t)j * dy;
      T yy = T(0);
      if (yy_col >= 0)
        for (int t = 0; t < d; ++t) yy += src[t] * src[t];
      for (int t = d; t < dy; ++t) dst[t] = (t == yy_col) ? yy : T(0);
    }
  if (pm) {                                         // Eq.rho numerator (X1)
    for (int h = 16; h >= 1; h >>= 1) racc += __shfl_xor_sync(0xffffffffu, racc, h);
    if (lane == 0) pm[s] = (double)mk * xs[d] + racc;
  }
  // weights: the simplex check (fp64, lane-strided then a butterfly) and the working-precision total
  // in sequential order like the oracle (every lane adds the shuffled values j = 0, 1, ... in turn)
  double sum = 0.0;
  T tot = T(0);
  for (int c0 = 0; c0 < mk; c0 += 32) {
    const T wv = (c0 + lane < mk) ? Wsrc[so + c0 + lane] : T(0);
    if (c0 + lane < mk) sum += (double)wv;
    const int n = mk - c0 < 32 ? mk - c0 : 32;
    for (int jj = 0; jj < n; ++jj) tot += __shfl_sync(0xffffffffu, wv, jj);
  }
  for (int h = 16; h >= 1; h >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, h);
  if (lane == 0 && !(fabs(sum - 1.0) <= wtol)) atomicOr(err, ERR_WEIGHTS);
  for (int j = lane; j < mk; j += 32) om[dsto + j] = Wsrc[so + j] / tot;
}

// per cluster: sum_i x_i (d values) and sum_i |x_i|^2 in fp64 (the Eq.rho numerator in k_gather)
template <typename T>
__global__ void k_xsums(const T* __restrict__ x, int m, int d, double* __restrict__ out) {
  const int c = blockIdx.x, lane = threadIdx.x;
  double q = 0.0;
  for (int t = lane; t < d; t += 32) {
    double sx = 0.0;
    for (int i = 0; i < m; ++i) {
      const double v = (double)x[((int64_t)c * m + i) * d + t];
      sx += v;
      q = fma(v, v, q);
    }
    out[(int64_t)c * (d + 1) + t] = sx;
  }
  for (int h = 16; h >= 1; h >>= 1) q += __shfl_xor_sync(0xffffffffu, q, h);
  if (lane == 0) out[(int64_t)c * (d + 1) + d] = q;
}

// Offset of entry (i, j) in a member's plan block (leading dimension ld >= m).  The column-major
// layout puts (i, j) at j ld + i; the "pair layout" of the variant-2 kernel with 32-row blocks
// interleaves columns 2q and 2q+1 by row ((i, 2q) at 2q ld + 2i, (i, 2q+1) at 2q ld + 2i + 1),
// so a lane moves both with one 8-byte access; an odd m_k's last column keeps j ld + i.  Both
// layouts fill exactly ld m_k elements per member.
__host__ __device__ __forceinline__ int64_t blk_idx(int i, int j, int mk, int ld, bool pair) {
  if (!pair || j >= (mk & ~1)) return (int64_t)j * ld + i;
  return (int64_t)(j & ~1) * ld + 2 * i + (j & 1);
}

// Pi^(2),0 = w_i w_j^(k) or, for warm members, the cached block;
// Lambda = 0.  Writes the new Pi2 into `dst` (a buffer distinct from the warm source).  The warm
// source keeps the previous round's block layout (ld_src rows, pair layout or not), which differs
// from this round's when the kernel variant changed (e.g. the largest m_k crossed 32).
template <typename T>
__global__ void __launch_bounds__(128)
k_init_plans(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
             const int32_t* __restrict__ item_cl, const int64_t* __restrict__ warm_src,
             const T* __restrict__ om, const T* __restrict__ w, const T* __restrict__ Qold,
             T* __restrict__ dst, T* __restrict__ L, int m, int ld, bool pair, int ld_src, bool pair_src) {
  const bool same = ld_src == ld && pair_src == pair;
  // warp per member, lane = row i (rows in chunks of 32), one column per step: coalesced rows
  const int item = blockIdx.x;
  const int c = item_cl[item];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t k = item_mb[item] + warp; k < item_mb[item + 1]; k += 4) {
    const int64_t o0 = off[k];
    const int mk = (int)(off[k + 1] - o0);
    const int64_t base = (int64_t)ld * o0;
    const int64_t src = warm_src ? warm_src[k] : -1;
    for (int r0 = 0; r0 < ld; r0 += 32) {
      const int i = r0 + lane;
      if (i >= ld) break;
      const T wi = i < m ? w[(int64_t)c * m + i] : T(0);
      int j = 0;
      if (pair)                                        // both columns of a pair per access
        for (; j + 1 < mk; j += 2) {
          const int64_t e = (int64_t)j * ld + 2 * i;
          typedef typename std::conditional<sizeof(T) == 4, float2, double2>::type T2;
          T2 v;
          if (src >= 0 && same) {
            v = *reinterpret_cast<const T2*>(Qold + src + e);
          } else if (src >= 0) {
            v.x = i < m ? Qold[src + blk_idx(i, j, mk, ld_src, pair_src)] : T(0);
            v.y = i < m ? Qold[src + blk_idx(i, j + 1, mk, ld_src, pair_src)] : T(0);
          } else {
            v.x = wi * om[o0 + j];
            v.y = wi * om[o0 + j + 1];
          }
          *reinterpret_cast<T2*>(dst + base + e) = v;
          T2 z;
          z.x = T(0);
          z.y = T(0);
          *reinterpret_cast<T2*>(L + base + e) = z;
        }
      for (; j < mk; ++j) {
        const int64_t e = blk_idx(i, j, mk, ld, pair);
        T q = wi * om[o0 + j];
        if (src >= 0) q = same ? Qold[src + e] : (i < m ? Qold[src + blk_idx(i, j, mk, ld_src, pair_src)] : T(0));
        dst[base + e] = q;
        L[base + e] = T(0);
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(128)
k_scatter_plans(const int32_t* __restrict__ order, const int64_t* __restrict__ off,
                const int64_t* __restrict__ orig_off, const T* __restrict__ src, T* __restrict__ dst,
                int64_t N, int m, int ld, const int32_t* __restrict__ mem_cl, const T* __restrict__ unscale,
                bool pair) {
  // unscale != nullptr: divide by unscale[cluster] (the pre-scaled Lambda of variant 2)
  const int64_t s = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= N) return;
  const int64_t k = order[s];
  const int mk = (int)(off[s + 1] - off[s]);
  const int64_t ne = (int64_t)m * mk;
  const T* a = src + (int64_t)ld * off[s];
  T* b = dst + (int64_t)m * orig_off[k];
  const T sc = unscale ? unscale[mem_cl[s]] : T(1);
  for (int64_t e = lane; e < ne; e += 32) {
    const int64_t j = e / m, i = e - j * m;
    const int64_t q = blk_idx((int)i, (int)j, mk, ld, pair);
    b[e] = unscale ? a[q] / sc : a[q];
  }
}

}  // namespace ad2k

namespace ad2k {
// ---------------------------------------------------------------------------------------------
// Device-side layout of a round (ad2_barycenter_init): validation + per-cluster histograms, a
// stable radix sort of the labels (CUB) gives the cluster-sorted member order, scans give the
// sorted offsets and the work-item table.  Only a handful of scalars come back to the host.
// scal[0]: error bits (1: offsets[0] != 0, 2: m_k < 1 or label out of range, 4: warm mismatch)
// scal[1]: max m_k    scal[2]: number of work items
// ---------------------------------------------------------------------------------------------
static __global__ void k_layout_hist(const int64_t* __restrict__ off, const int32_t* __restrict__ lab, int64_t N,
                                     int K, int32_t* __restrict__ keys, int32_t* __restrict__ iota,
                                     unsigned long long* __restrict__ cnt, unsigned long long* __restrict__ pts,
                                     unsigned long long* __restrict__ scal) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0 && off[0] != 0) atomicOr(&scal[0], 1ull);
  unsigned mk32 = 0;
  if (k < N) {
    const int64_t mk = off[k + 1] - off[k];
    int l = lab[k];
    const bool bad = mk < 1 || mk > 0x7fffffff || l < 0 || l >= K;
    if (bad) {
      atomicOr(&scal[0], 2ull);
      l = 0;
    } else {
      atomicAdd(&cnt[l], 1ull);
      atomicAdd(&pts[l], (unsigned long long)mk);
      mk32 = (unsigned)mk;
    }
    keys[k] = l;
    iota[k] = (int32_t)k;
  }
  const unsigned wmax = __reduce_max_sync(0xffffffffu, mk32);
  if ((threadIdx.x & 31) == 0 && wmax > 0) atomicMax(&scal[1], (unsigned long long)wmax);
}

static __global__ void k_layout_sorted(const int32_t* __restrict__ order, const int64_t* __restrict__ off_in,
                                       int64_t N, int64_t* __restrict__ sz, int64_t* __restrict__ pos_of) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < N) {
    const int64_t k = order[s];
    sz[s] = off_in[k + 1] - off_in[k];
    pos_of[k] = s;
  } else if (s == N) {
    sz[N] = 0;
  }
}

static __global__ void k_layout_items_count(const unsigned long long* __restrict__ cnt, int K, int64_t per_item,
                                            int64_t* __restrict__ cstart, int64_t* __restrict__ cl_item,
                                            unsigned long long* __restrict__ scal) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t acc = 0, it = 0;
  for (int c = 0; c < K; ++c) {
    cstart[c] = acc;
    cl_item[c] = it;
    acc += (int64_t)cnt[c];
    it += ((int64_t)cnt[c] + per_item - 1) / per_item;
  }
  cstart[K] = acc;
  cl_item[K] = it;
  scal[2] = (unsigned long long)it;
}

static __global__ void k_layout_items_fill(const int64_t* __restrict__ cstart, const int64_t* __restrict__ cl_item,
                                           int K, int64_t per_item, int64_t N, int64_t* __restrict__ item_mb,
                                           int32_t* __restrict__ item_cl) {
  const int c = blockIdx.x;
  for (int64_t it = cl_item[c] + threadIdx.x; it < cl_item[c + 1]; it += blockDim.x) {
    item_mb[it] = cstart[c] + (it - cl_item[c]) * per_item;
    item_cl[it] = c;
  }
  if (c == K - 1 && threadIdx.x == 0) item_mb[cl_item[K]] = N;
}

static __global__ void k_layout_warm(const int32_t* __restrict__ order, const uint8_t* __restrict__ warm,
                                     const int64_t* __restrict__ pos_old, const int64_t* __restrict__ off_old,
                                     int64_t N_old, int ld_old, const int64_t* __restrict__ off_new, int64_t N,
                                     int64_t* __restrict__ warm_src, unsigned long long* __restrict__ scal) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= N) return;
  const int64_t k = order[s];
  if (!warm[k]) {
    warm_src[s] = -1;
    return;
  }
  if (k >= N_old) {
    atomicOr(&scal[0], 4ull);
    warm_src[s] = -1;
    return;
  }
  const int64_t ps = pos_old[k];
  if (off_old[ps + 1] - off_old[ps] != off_new[s + 1] - off_new[s]) {
    atomicOr(&scal[0], 4ull);
    warm_src[s] = -1;
    return;
  }
  warm_src[s] = (int64_t)ld_old * off_old[ps];
}
}  // namespace ad2k

namespace ad2k {
// member cluster of each sorted member (from the work-item table)
static __global__ void k_member_cluster(const int64_t* __restrict__ item_mb, const int32_t* __restrict__ item_cl,
                                        int64_t n_items, int32_t* __restrict__ mem_cl) {
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  for (int64_t s = item_mb[it]; s < item_mb[it + 1]; ++s) mem_cl[s] = item_cl[it];
}

// Symbolic supports: member symbol ids into the sorted layout, and the cost from the
// table, C_ij = D[xs_i, ys_j] (cached; rows >= m are 0) with optional per-item sums for rho.
// err bit ERR_SYMBOL: an id outside [0, V).
constexpr int ERR_SYMBOL = 4;
static __global__ void k_gather_sym(const int32_t* __restrict__ order, const int64_t* __restrict__ src_off,
                                    const int64_t* __restrict__ dst_off, const int32_t* __restrict__ ys_src,
                                    int32_t* __restrict__ ys, int64_t N) {
  const int64_t s = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= N) return;
  const int64_t k = order[s];
  const int64_t so = src_off[k], dsto = dst_off[s];
  const int mk = (int)(src_off[k + 1] - so);
  for (int j = lane; j < mk; j += 32) ys[dsto + j] = ys_src[so + j];
}

template <typename T>
__global__ void __launch_bounds__(128)
k_cost_table(const int64_t* __restrict__ off, const int64_t* __restrict__ item_mb,
             const int32_t* __restrict__ item_cl, const int32_t* __restrict__ ys, const int32_t* __restrict__ xs,
             const T* __restrict__ D, int V, T* __restrict__ Cc, double* __restrict__ psum, int m, int ld, int* err) {
  const int item = blockIdx.x;
  const int c = item_cl[item];
  const int64_t p0 = off[item_mb[item]], p1 = off[item_mb[item + 1]];
  double acc = 0.0;
  bool bad = false;
  for (int64_t e = (int64_t)threadIdx.x; e < (p1 - p0) * ld; e += blockDim.x) {
    const int64_t p = e / ld;
    const int i = (int)(e - p * ld);
    T v = T(0);
    if (i < m) {
      const int a = xs[(int64_t)c * m + i], b = ys[p0 + p];
      if (a < 0 || a >= V || b < 0 || b >= V) bad = true;
      else v = D[(int64_t)a * V + b];
    }
    Cc[ld * p0 + e] = v;
    acc += (double)v;
  }
  if (bad) atomicOr(err, ERR_SYMBOL);
  if (psum) {
    for (int h = 16; h >= 1; h >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, h);
    __shared__ double sh[4];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) psum[item] = (sh[0] + sh[1]) + (sh[2] + sh[3]);
  }
}

// per-cluster sum of per-member doubles over the cluster's sorted members [cstart[c], cstart[c+1]):
// fixed strided order per thread, then a fixed-shape tree -> deterministic
static __global__ void k_dsum_members(const double* __restrict__ pm, const int64_t* __restrict__ cstart,
                                      double* __restrict__ S) {
  const int c = blockIdx.x;
  __shared__ double red[256];
  double a = 0.0;
  for (int64_t s = cstart[c] + threadIdx.x; s < cstart[c + 1]; s += 256) a += pm[s];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int h = 128; h >= 1; h >>= 1) {
    if ((int)threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) S[c] = red[0];
}
}  // namespace ad2k
