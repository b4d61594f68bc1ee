// ad2_seed.cu — the initial partition of AD2-clustering on the GPU:
// k-means++ D^2 seeding and Lloyd iterations on sampled member means, every member labelled to its
// nearest mean with the empty-cluster repair, and the member picked per cluster for Eq.merge.
//
// Alg. 1 starts from "K random centroid[s]"; the recipe is SURVEY.md §8(d)'s (k-means++,
// the paper's comparison method; a random member with >= m support points).
// Every random draw is an input (sample indices, uniforms), the readings that turn a draw into an
// index are DESIGN.md X20-X23.  Everything is fp64; every sum that decides an index has a fixed
// order:
//   - a squared distance is sum_t (p_t - c_t)^2 in coordinate order with the multiply and the add
//     rounded separately (__dmul_rn / __dadd_rn: no contraction into FMA), so it is the same
//     number on any device or host that evaluates the same expression (X21);
//   - a member mean sum_j w_j y_j is accumulated over j in order (lane per coordinate);
//   - a Lloyd centre is the sum of its points in index order (one warp per cluster walks the
//     labels in order, lane per coordinate) divided by the count;
//   - the D^2 draw (X20) sums D^2 in 256-point blocks (fixed tree) and scans the block sums and
//     then the chosen block with a fixed two-level order.  This order differs from a sequential
//     prefix by rounding only, so the drawn index can differ only when u * sum D^2 falls within
//     rounding of a prefix boundary (X20).
// No float atomics anywhere; counts are integer atomics.
#include <cuda_runtime.h>
#include <stdint.h>

namespace ad2s {

constexpr int SEED_BLK = 256;     // points per D^2 block sum

__device__ __forceinline__ double sqd(const double* __restrict__ p, const double* __restrict__ c, int d) {
  double acc = 0.0;
  for (int t = 0; t < d; ++t) {
    const double df = __dsub_rn(p[t], c[t]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  return acc;
}

// mu[r][t] = sum_j w_j y_jt of member idx[r] (idx == nullptr: member r); warp per row, lane per t
template <typename T>
__global__ void k_member_means(const int64_t* __restrict__ off, const T* __restrict__ Y, const T* __restrict__ W,
                               const int64_t* __restrict__ idx, int64_t rows, int d, double* __restrict__ mu) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int64_t k = idx ? idx[r] : r;
  const int64_t a = off[k], e = off[k + 1];
  for (int t = lane; t < d; t += 32) {
    double acc = 0.0;
    for (int64_t j = a; j < e; ++j) acc = __dadd_rn(acc, __dmul_rn((double)W[j], (double)Y[j * d + t]));
    mu[r * d + t] = acc;
  }
}

// D^2 after centre c: d2[i] = min(d2[i], |P_i - centre|^2) (first: = the distance), and the
// 256-point block sums of d2 by a fixed tree
__global__ void k_d2_update(const double* __restrict__ P, int64_t ns, int d, const double* __restrict__ centre,
                            int first, double* __restrict__ d2, double* __restrict__ bsum) {
  __shared__ double red[SEED_BLK];
  const int64_t i = (int64_t)blockIdx.x * SEED_BLK + threadIdx.x;
  double v = 0.0;
  if (i < ns) {
    const double nd = sqd(P + i * d, centre, d);
    v = first ? nd : fmin(d2[i], nd);
    d2[i] = v;
  }
  red[threadIdx.x] = v;
  __syncthreads();
  for (int s = SEED_BLK / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = red[0];
}

// warp-level first crossing: lanes own contiguous chunks of v[0..n); returns the first index whose
// inclusive prefix (base + earlier chunks' sums + in-chunk prefix) exceeds target, or -1;
// *run_end = base + the total, *before = the prefix just before the returned index (all lanes)
__device__ int64_t warp_first_crossing(const double* __restrict__ v, int64_t n, double base, double target,
                                       double* run_end, double* before) {
  const int lane = threadIdx.x & 31;
  const int64_t per = (n + 31) / 32;
  const int64_t a = lane * per, e = a + per < n ? a + per : n;
  double cs = 0.0;
  for (int64_t i = a; i < e; ++i) cs = __dadd_rn(cs, v[i]);
  // exclusive prefix of the chunk sums in lane order (sequential over lanes: fixed order)
  double excl = base;
  for (int l = 0; l < 32; ++l) {
    const double s = __shfl_sync(0xffffffffu, cs, l);
    if (l < lane) excl = __dadd_rn(excl, s);
  }
  const double incl = __dadd_rn(excl, cs);
  *run_end = __shfl_sync(0xffffffffu, incl, 31);
  const unsigned hit = __ballot_sync(0xffffffffu, a < e && incl > target);
  if (!hit) return -1;
  const int L = __ffs(hit) - 1;
  int64_t found = -1;
  double bef = excl;
  if (lane == L) {
    double run = excl;
    for (int64_t i = a; i < e; ++i) {
      const double nx = __dadd_rn(run, v[i]);
      if (nx > target) {
        found = i;
        bef = run;
        break;
      }
      run = nx;
    }
    if (found < 0) {                    // the chunk sum crossed, its prefix scan fell short by rounding
      found = e - 1;
      bef = __dsub_rn(run, v[e - 1]);
    }
  }
  *before = __shfl_sync(0xffffffffu, bef, L);
  return __shfl_sync(0xffffffffu, found, L);
}

// last index in [a, e) with v > 0, or -1 (one warp)
__device__ int64_t warp_last_positive(const double* __restrict__ v, int64_t a, int64_t e) {
  int64_t last = -1;
  for (int64_t q = a + (threadIdx.x & 31); q < e; q += 32)
    if (v[q] > 0.0) last = q;
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t t = __shfl_xor_sync(0xffffffffu, last, o);
    last = t > last ? t : last;
  }
  return last;
}

// the D^2 draw of centre c (X20): one warp.  total = fixed-order sum of the block sums; the first
// block whose inclusive block prefix exceeds u * total, then the first point inside it whose
// prefix (continuing from the block's exclusive prefix) exceeds it; a point with D^2 = 0 is never
// drawn (rounding fall-backs: the block's, else the sample's, last point with D^2 > 0).
// total = 0: sample point floor(u * ns).  Writes centre c = P[i].
__global__ void k_d2_select(const double* __restrict__ P, int64_t ns, int d, const double* __restrict__ d2,
                            const double* __restrict__ bsum, int64_t nb, double u, double* __restrict__ centre,
                            int64_t* __restrict__ chosen) {
  double total, ex, dummy;
  warp_first_crossing(bsum, nb, 0.0, INFINITY, &total, &dummy);
  int64_t i = -1;
  if (total > 0.0) {
    const double target = __dmul_rn(u, total);
    const int64_t b = warp_first_crossing(bsum, nb, 0.0, target, &dummy, &ex);
    if (b >= 0) {
      const int64_t a = b * SEED_BLK;
      const int64_t n = ns - a < SEED_BLK ? ns - a : SEED_BLK;
      const int64_t j = warp_first_crossing(d2 + a, n, ex, target, &dummy, &dummy);
      if (j >= 0 && d2[a + j] > 0.0) i = a + j;
      else i = warp_last_positive(d2, a, a + n);
    }
    if (i < 0) i = warp_last_positive(d2, 0, ns);
  } else {
    i = (int64_t)(u * (double)ns);
    if (i > ns - 1) i = ns - 1;
  }
  for (int t = threadIdx.x & 31; t < d; t += 32) centre[t] = P[i * d + t];
  if ((threadIdx.x & 31) == 0 && chosen) *chosen = i;
}

// nearest centre of every point (ties: lowest index), optional integer counts
__global__ void k_nearest(const double* __restrict__ P, int64_t n, int d, const double* __restrict__ cen, int K,
                          int32_t* __restrict__ lab, int* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* p = P + i * d;
  double best = sqd(p, cen, d);
  int bc = 0;
  for (int c = 1; c < K; ++c) {
    const double v = sqd(p, cen + (size_t)c * d, d);
    if (v < best) {
      best = v;
      bc = c;
    }
  }
  lab[i] = bc;
  if (counts) atomicAdd(counts + bc, 1);
}

// Lloyd centre: warp per cluster, labels walked in index order (4 per lane per load, the next load
// issued before the current one is consumed), lane per coordinate (d <= 32 * DQ); an empty cluster
// keeps its centre
template <int DQ>
__global__ void k_lloyd_centres(const double* __restrict__ P, int64_t n, int d, const int32_t* __restrict__ lab,
                                int K, double* __restrict__ cen) {
  const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= K) return;
  double acc[DQ];
#pragma unroll
  for (int q = 0; q < DQ; ++q) acc[q] = 0.0;
  int64_t cnt = 0;
  const int64_t n4 = n & ~(int64_t)127;
  int4 nxt = make_int4(-1, -1, -1, -1);
  if (n4 > 0) nxt = reinterpret_cast<const int4*>(lab)[lane];
  for (int64_t base = 0; base < n; base += 128) {
    int l4[4];
    if (base < n4) {
      l4[0] = nxt.x, l4[1] = nxt.y, l4[2] = nxt.z, l4[3] = nxt.w;
      if (base + 128 < n4) nxt = reinterpret_cast<const int4*>(lab + base + 128)[lane];
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t i = base + 4 * lane + q;
        l4[q] = i < n ? lab[i] : -1;
      }
    }
    const unsigned nib = (l4[0] == c) | ((l4[1] == c) << 1) | ((l4[2] == c) << 2) | ((l4[3] == c) << 3);
    unsigned any = __ballot_sync(0xffffffffu, nib != 0);
    while (any) {
      const int L = __ffs(any) - 1;
      any &= any - 1;
      unsigned bits = __shfl_sync(0xffffffffu, nib, L);
      while (bits) {
        const int q = __ffs(bits) - 1;
        bits &= bits - 1;
        const int64_t i = base + 4 * L + q;
#pragma unroll
        for (int r = 0; r < DQ; ++r) {
          const int t = lane + 32 * r;
          if (t < d) acc[r] = __dadd_rn(acc[r], P[i * d + t]);
        }
        ++cnt;
      }
    }
  }
  if (cnt > 0) {
#pragma unroll
    for (int r = 0; r < DQ; ++r) {
      const int t = lane + 32 * r;
      if (t < d) cen[(size_t)c * d + t] = __ddiv_rn(acc[r], (double)cnt);
    }
  }
}

// empty-cluster repair (X22): the member farthest from its own centre among clusters with >= 2
// members (others count -1), first index on ties; per-block (value, index), then one block
struct VI {
  double v;
  int64_t i;
};
__device__ __forceinline__ VI vi_max(VI a, VI b) { return (b.v > a.v || (b.v == a.v && b.i < a.i)) ? b : a; }

__global__ void k_far_blocks(const double* __restrict__ mu, int64_t N, int d, const int32_t* __restrict__ lab,
                             const double* __restrict__ cen, const int* __restrict__ counts, VI* __restrict__ out) {
  __shared__ VI red[256];
  VI best{-INFINITY, INT64_MAX};
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < N; i += (int64_t)gridDim.x * 256) {
    const int e = lab[i];
    const double v = counts[e] <= 1 ? -1.0 : sqd(mu + i * d, cen + (size_t)e * d, d);
    best = vi_max(best, VI{v, i});
  }
  red[threadIdx.x] = best;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = vi_max(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = red[0];
}

__global__ void k_far_final(const VI* __restrict__ part, int nb, int64_t* __restrict__ k_out) {
  __shared__ VI red[256];
  VI best{-INFINITY, INT64_MAX};
  for (int b = threadIdx.x; b < nb; b += 256) best = vi_max(best, part[b]);
  red[threadIdx.x] = best;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = vi_max(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *k_out = red[0].i;
}

// move member k to cluster c: labels, counts, centre c = mu_k (one warp)
__global__ void k_repair_move(const double* __restrict__ mu, int d, const int64_t* __restrict__ kp, int c,
                              int32_t* __restrict__ lab, int* __restrict__ counts, double* __restrict__ cen) {
  const int64_t k = *kp;
  const int lane = threadIdx.x & 31;
  for (int t = lane; t < d; t += 32) cen[(size_t)c * d + t] = mu[k * d + t];
  if (lane == 0) {
    counts[lab[k]] -= 1;
    counts[c] += 1;
    lab[k] = c;
  }
}

// X23: warp per cluster; position floor(u_c * n_big) among the members with m_k >= m in index
// order, else the first member with the largest m_k; -1 for an empty cluster
__global__ void k_pick_members(const int64_t* __restrict__ off, const int32_t* __restrict__ lab, int64_t N, int m,
                               const double* __restrict__ u, int K, int64_t* __restrict__ pick) {
  const int c = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= K) return;
  int64_t nbig = 0, bestk = -1, bestmk = -1;
  for (int64_t b = 0; b < N; b += 32) {
    const int64_t k = b + lane;
    const bool in = k < N && lab[k] == c;
    const int64_t mk = in ? off[k + 1] - off[k] : -1;
    nbig += __popc(__ballot_sync(0xffffffffu, in && mk >= m));
    // first member with the largest m_k: max m_k, then lowest index
    int64_t vm = mk, vk = in ? k : INT64_MAX;
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t om = __shfl_xor_sync(0xffffffffu, vm, o), ok = __shfl_xor_sync(0xffffffffu, vk, o);
      if (om > vm || (om == vm && ok < vk)) vm = om, vk = ok;
    }
    if (vm > bestmk) bestmk = vm, bestk = vk;
  }
  int64_t res = bestk;
  if (nbig > 0) {
    int64_t want = (int64_t)(u[c] * (double)nbig);
    if (want > nbig - 1) want = nbig - 1;
    int64_t seen = 0;
    res = -1;
    for (int64_t b = 0; b < N && res < 0; b += 32) {
      const int64_t k = b + lane;
      const bool big = k < N && lab[k] == c && off[k + 1] - off[k] >= m;
      const unsigned bal = __ballot_sync(0xffffffffu, big);
      const int nb = __popc(bal);
      if (seen + nb > want) {
        unsigned bits = bal;
        for (int64_t s = seen; s < want; ++s) bits &= bits - 1;
        res = b + __ffs(bits) - 1;
      }
      seen += nb;
    }
  }
  if (lane == 0) pick[c] = res;
}

}  // namespace ad2s

// ---- launchers (called from ad2.cu) ----------------------------------------------------------
using namespace ad2s;

int seed_blk() { return SEED_BLK; }

void seed_means_launch(int f64, const int64_t* off, const void* Y, const void* W, const int64_t* idx, int64_t rows,
                       int d, double* mu, cudaStream_t s) {
  if (rows <= 0) return;
  const unsigned g = (unsigned)((rows * 32 + 255) / 256);
  if (f64)
    k_member_means<double><<<g, 256, 0, s>>>(off, (const double*)Y, (const double*)W, idx, rows, d, mu);
  else
    k_member_means<float><<<g, 256, 0, s>>>(off, (const float*)Y, (const float*)W, idx, rows, d, mu);
}

void seed_d2_launch(const double* P, int64_t ns, int d, const double* centre, int first, double* d2, double* bsum,
                    cudaStream_t s) {
  k_d2_update<<<(unsigned)((ns + SEED_BLK - 1) / SEED_BLK), SEED_BLK, 0, s>>>(P, ns, d, centre, first, d2, bsum);
}

void seed_select_launch(const double* P, int64_t ns, int d, const double* d2, const double* bsum, double u,
                        double* centre, int64_t* chosen, cudaStream_t s) {
  k_d2_select<<<1, 32, 0, s>>>(P, ns, d, d2, bsum, (ns + SEED_BLK - 1) / SEED_BLK, u, centre, chosen);
}

void seed_nearest_launch(const double* P, int64_t n, int d, const double* cen, int K, int32_t* lab, int* counts,
                         cudaStream_t s) {
  if (n <= 0) return;
  k_nearest<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(P, n, d, cen, K, lab, counts);
}

void seed_lloyd_launch(const double* P, int64_t n, int d, const int32_t* lab, int K, double* cen, cudaStream_t s) {
  const unsigned g = (unsigned)((K * 32 + 127) / 128);
  if (d <= 32) k_lloyd_centres<1><<<g, 128, 0, s>>>(P, n, d, lab, K, cen);
  else if (d <= 64) k_lloyd_centres<2><<<g, 128, 0, s>>>(P, n, d, lab, K, cen);
  else if (d <= 128) k_lloyd_centres<4><<<g, 128, 0, s>>>(P, n, d, lab, K, cen);
  else k_lloyd_centres<8><<<g, 128, 0, s>>>(P, n, d, lab, K, cen);
}

size_t seed_far_scratch() { return sizeof(VI) * 1024 + sizeof(int64_t); }

void seed_repair_launch(const double* mu, int64_t N, int d, int32_t* lab, double* cen, int* counts, int c,
                        void* scratch, cudaStream_t s) {
  VI* part = static_cast<VI*>(scratch);
  int64_t* kp = reinterpret_cast<int64_t*>(part + 1024);
  int nb = (int)((N + 255) / 256);
  if (nb > 1024) nb = 1024;
  k_far_blocks<<<nb, 256, 0, s>>>(mu, N, d, lab, cen, counts, part);
  k_far_final<<<1, 256, 0, s>>>(part, nb, kp);
  k_repair_move<<<1, 32, 0, s>>>(mu, d, kp, c, lab, counts, cen);
}

void seed_pick_launch(const int64_t* off, const int32_t* lab, int64_t N, int m, const double* u, int K, int64_t* pick,
                      cudaStream_t s) {
  k_pick_members<<<(unsigned)((K * 32 + 127) / 128), 128, 0, s>>>(off, lab, N, m, u, K, pick);
}
