/*
 * ad2.h — C ABI of libad2: the modified Bregman-ADMM Wasserstein-barycenter update of
 * AD2-clustering (Ye, Wu, Wang, Li; arXiv 1510.00012, Algorithm 4) on NVIDIA B200 (sm_100a).
 *
 * "P:n" = PAPER.md line n (the paper's LaTeX source); equations are named by their LaTeX
 * label (the PDF numbers them (1)-(24), SURVEY.md §0 has the map).
 *
 * Problem.  N members P^(k) = {(w_j^(k), x_j^(k)), j = 1..m_k} in R^d, each with a
 * cluster label l^(k) in [0, K).  For every cluster c the library keeps a centroid
 * P_c = {(w_i, x_i), i = 1..m} and the B-ADMM state of each member: Pi^(k,1), Pi^(k,2),
 * Lambda^(k) in R^{m x m_k}, and runs Alg. 4:
 *
 *   init            : C^(k) = (||x_i - x_j^(k)||^2)_ij; rho_c = rho0 * mean_{k in c,i,j} C_ij
 *                     (Eq.rho, reading X1); Lambda = 0; Pi^(k,2) = w_i w_j^(k)
 *                      or the cached Pi^(k,2) for warm members
 *   step (1 iter)   : Pi^(k,1) (Eq.badmmc0b, Eq.badmmc0); pt^(k,1) (Eq.badmmc1b);
 *                     w by R1 (Eq.badmmw) or R2 (Eq.badmmw2) — a reduction
 *                     over all members of the cluster, on all ranks; Pi^(k,2) (Eq.badmmc1);
 *                     Lambda += rho (Pi^(k,1) - Pi^(k,2)) (Eq.badmm2)
 *   update_support  : x_i = sum_k sum_j pi2_ij x_j^(k) / sum_k sum_j pi2_ij (Eq.updatex, P:342-351,
 *                     readings X5, X12), then C is rebuilt; rho stays fixed (X2)
 *   objective       : F_c = (1/N_c) sum_{k in c} <C^(k), Pi^(k,1)> (X14)
 *
 * The caller drives the schedule of Alg. 4: for e in 1..T/tau: step(tau); update_support().
 *
 * Conventions
 *  - All calls are made from one host thread per context; a context is NOT thread-safe.
 *  - Compute is asynchronous on the context's CUDA stream (the stream given to ad2_create).
 *    Calls that return host data (init, objective, getters with AD2_HOST, sync) synchronise it.
 *  - Argument errors are detected before any state changes and return AD2_ERR_ARG.
 *    Device-side faults (a non-finite plan/weight) are latched and returned by the next
 *    synchronising call as AD2_ERR_NONFINITE.  No C++ exception crosses this ABI.
 *  - There is no CPU fallback: without a CUDA device ad2_create returns AD2_ERR_CUDA.
 *  - Floating-point buffers are float (AD2_F32) or double (AD2_F64) per the batch dtype.
 *    eps is params->eps in both precisions (reading X3).
 *  - Multi-GPU: one context per GPU/process, each with its own member shard; every
 *    rank calls every function with the same d, m, K, params, x0, w0 and the same schedule.
 *    The per-cluster partial sums (w: K*m per iteration, x: K*m*(d+1) per support update, rho
 *    and objective: K) are summed across ranks by NCCL all-reduce over NVLink (or by a host
 *    process group, below).  Errors agree across ranks: ad2_barycenter_init, ad2_objective,
 *    ad2_sync and ad2_cluster exchange every rank's status before the next collective, so a
 *    rank-local error (a bad label, weights off the simplex, a non-finite value) makes every
 *    rank return an error instead of leaving the others waiting in a collective.  A rank with
 *    no members (n_members = 0) takes part in every collective with zero partial sums.
 */
#ifndef AD2_H
#define AD2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AD2_ABI_VERSION 3

typedef struct ad2_ctx_s *ad2_ctx;

typedef enum { AD2_F32 = 0, AD2_F64 = 1 } ad2_dtype;
typedef enum { AD2_R1 = 0, AD2_R2 = 1 } ad2_rule;          /* Eq.badmmw / Eq.badmmw2 */
typedef enum { AD2_DEVICE = 0, AD2_HOST = 1 } ad2_mem;     /* where a caller buffer lives */
typedef enum { AD2_PI1 = 0, AD2_PI2 = 1, AD2_LAMBDA = 2, AD2_COST = 3 } ad2_plan;
/* Cost build for the cached-cost kernels (m > 32, m_k > 32 or d > 16):
 *  AD2_COST_FP32   : fp32 FMAs, C = |x|^2 + |y|^2 - 2 x.y clamped at 0 (the parity default);
 *  AD2_COST_TC_BF16: tcgen05 tensor cores, x and y rounded to bf16, fp32 accumulation in TMEM;
 *                    |dC| <= 2^-7 |x_i||y_j| (+ fp32 rounding).  SURVEY.md §8(d) config 4.
 *                    AD2_ERR_ARG when the round does not use the cached-cost warp-pair kernel.
 * (m <= 32 with d <= 16 recomputes C in fp32 inside the iteration kernel; cost_mode must be 0.) */
typedef enum { AD2_COST_FP32 = 0, AD2_COST_TC_BF16 = 1, AD2_COST_TABLE = 2 } ad2_cost_mode;
/* AD2_COST_TABLE: symbolic supports — the support points are symbols of a fixed set
 * with a symbol-to-symbol cost table D (ad2_set_cost_table): batch->d must be 1, batch->supports
 * and x0 hold int32 symbol ids ([n] and [K][m]), C^(k)_ij = D[x_i][y_j], the support update is
 * skipped (ad2_update_support is a no-op), ad2_get_centroids returns the int32 ids in x.  Runs
 * on the cached-cost kernels (variant 3 for fp32 with m, m_k <= 64, else the generic one). */

typedef enum {
    AD2_OK = 0,
    AD2_ERR_ARG = 1,        /* bad argument (shape, pointer, offsets, label range, weights off the simplex) */
    AD2_ERR_OOM = 2,        /* device allocation failed */
    AD2_ERR_CUDA = 3,       /* CUDA runtime error (message in ad2_last_error) */
    AD2_ERR_NCCL = 4,       /* NCCL error or NCCL unavailable */
    AD2_ERR_NONFINITE = 5,  /* a plan row mass / weight became non-finite (latched, async) */
    AD2_ERR_ZERO_RHO = 6,   /* a cluster's mean cost is 0 (rho = 0) */
    AD2_ERR_EMPTY = 7,      /* a cluster has no members on any rank */
    AD2_ERR_STATE = 8       /* call out of order (e.g. step before init) */
} ad2_status;

/* One rank's member shard in the paper's ragged layout.  Borrowed, read-only,
 * only during ad2_barycenter_init (the library copies what it needs). */
typedef struct {
    ad2_dtype dtype;
    ad2_mem mem;                /* where offsets/supports/weights/labels (and x0/w0) live */
    int32_t d;                  /* support dimension, >= 1 */
    int32_t m;                  /* centroid support size, >= 1 */
    int32_t K;                  /* number of clusters, >= 1 */
    int64_t n_members;          /* N on this rank, >= 0 */
    const int64_t *offsets;     /* [N+1], offsets[0] = 0, m_k = offsets[k+1]-offsets[k] >= 1 */
    const void *supports;       /* [offsets[N]][d] row-major: x_j^(k) = supports[offsets[k]+j] */
    const void *weights;        /* [offsets[N]]: w^(k) on the simplex, |sum - 1| <= 1e-6 (f64) or
                                   1e-5 (f32); renormalised by its sum (O1) */
    const int32_t *labels;      /* [N], each in [0, K) */
} ad2_batch;

typedef struct {
    double rho0;                /* > 0; rho_c = rho0 * mean cost of cluster c (X1); paper default 2 */
    double eps;                 /* >= 0; floor of Eq.badmmc0b / Eq.badmmc1b, paper 1e-16 */
    int32_t rule;               /* AD2_R1 or AD2_R2 */
    int32_t cost_mode;          /* ad2_cost_mode: how C is built when it is cached (see below) */
} ad2_params;

typedef struct {
    int32_t abi_version;
    int32_t dtype, d, m, K;
    int64_t n_members;          /* on this rank */
    int64_t n_points;           /* sum_k m_k on this rank */
    int64_t entries;            /* sum_k m * m_k on this rank (plan entries per iteration) */
    int64_t n_items;            /* work items (per-cluster member chunks) */
    int32_t variant;            /* 2 = TMA-staged fused kernel, cost recomputed in-kernel (m <= 32, d <= 16);
                                   3 = TMA-staged warp / warp-pair / warp-quad kernel with a cost cache (fp32,
                                   m <= 128, m_k <= 128, any d; configs 4 and symbolic rounds);
                                   0 = generic one-thread-per-member kernels (anything else) */
    int32_t mp, nch;            /* fused-kernel row tile (8/16/32) and column chunks */
    int32_t nranks, rank;
    int64_t launches;           /* kernels launched by this context so far (graph nodes counted) */
    int64_t state_bytes;        /* device bytes owned by the context */
    int32_t state_mode;         /* ad2_set_state_mode */
    int32_t eps_floor_columns;  /* 1: a compressed-state pass met a column whose mass is the eps floor's
                                   (the eps-free recursion does not hold there; use state mode 0) */
    int64_t assign_certified;   /* last ad2_cluster: member-rounds whose label the bounds certified (no solve) */
    int64_t assign_exact;       /* last ad2_cluster: exact transport solves (incl. the centroid drifts) */
    int32_t tc_cost;            /* 1: the iteration kernel forms the cost's dot products on the tensor
                                   cores (ad2_set_tc_cost and the round's shape allow it) */
} ad2_info;

/* Create a context on CUDA device `cuda_device`; `cuda_stream` is a cudaStream_t (NULL = legacy
 * default stream) that every later call enqueues on.  out receives the handle. */
ad2_status ad2_create(ad2_ctx *out, int cuda_device, void *cuda_stream);

/* Fill `id_out` (128 bytes, an ncclUniqueId) on one rank, to be broadcast by the caller (e.g.
 * through torch.distributed) before ad2_attach_nccl.  Returns AD2_ERR_NCCL if libnccl.so.2
 * cannot be loaded. */
ad2_status ad2_nccl_unique_id(void *id_out);

/* Join an NCCL communicator of `nranks` ranks (this one is `rank`), created from `unique_id`.
 * Must precede ad2_barycenter_init.  nranks == 1 is allowed (all-reduce degenerates to a copy). */
ad2_status ad2_attach_nccl(ad2_ctx ctx, int nranks, int rank, const void *unique_id);

/* ---- Host process group: the same cross-rank sums without NCCL --------------------------------
 * The member-sharded path needs one all-reduce of per-cluster
 * partial sums per iteration / support update / round.  NCCL needs one GPU per rank; a host
 * process group serves ranks that are processes on ONE host, e.g. several ranks sharing one GPU
 * (testing the sharded path on a one-GPU box) or hosts without NCCL.  Ranks share a POSIX
 * shared-memory segment `name` ("/..."); an all-reduce sums the ranks' buffers in rank order, so
 * every rank receives the bit-identical sum.  Inside libad2 it runs as a device->host copy, a
 * host-function node and a host->device copy in the step's CUDA graph (no kernel waits on
 * another rank).  A barrier that waits longer than AD2_GROUP_TIMEOUT seconds (default 300)
 * latches a failure: every later libad2 call on an attached context returns AD2_ERR_NCCL.
 *
 * ad2_group_open: collective over the `nranks` processes (blocks until all have joined);
 *   slot_bytes = the largest single all-reduce (>= 8 K m (d + 1) bytes covers libad2's use).
 * ad2_group_allreduce: in-place sum of `count` host elements (dtype AD2_GROUP_*) over the group.
 * ad2_attach_group: the context borrows g (g must outlive the context); instead of
 *   ad2_attach_nccl, before ad2_barycenter_init.
 * ad2_group_close: unmaps; call after every context using g is destroyed. */
typedef struct ad2_group_s *ad2_group;
enum { AD2_GROUP_F32 = 0, AD2_GROUP_F64 = 1, AD2_GROUP_U64 = 2 };
ad2_status ad2_group_open(ad2_group *out, const char *name, int nranks, int rank, int64_t slot_bytes);
ad2_status ad2_group_allreduce(ad2_group g, void *host_buf, int64_t count, int32_t dtype);
ad2_status ad2_attach_group(ad2_ctx ctx, ad2_group g);
void ad2_group_close(ad2_group g);

/* State representation of the iteration kernel (variant 2, steps of >= 3 iterations):
 *   0 (default): Pi1 and Lambda stream through HBM every iteration (16 B per plan entry in fp32),
 *     Alg. 4 exactly as written.
 *   1: epoch-anchored compressed state.  With the eps of
 *     Eq.badmmc0b / Eq.badmmc1b dropped from the Pi2 recursion, Lambda cancels between them and
 *     Pi2^t = G exp(-s C / rho) a_i b_j from an anchor G = Pi2^{t0} (pin P4).  Inside a step the
 *     passes stream G (read-only), U = Lambda + rho Pi1 and per-member log-factors: 12 B per
 *     entry instead of 16.  The first pass of a step forms G exactly (with eps) and the last pass
 *     stores Pi1 and Lambda again, so everything outside a step (read-back, objective, warm
 *     start) is unchanged.  Entries whose value is decided by eps differ (they keep decaying
 *     below the floor instead of sitting on it); a column whose whole mass is the floor's raises
 *     ad2_info.eps_floor_columns.
 * Takes effect at the next ad2_badmm_step. */
ad2_status ad2_set_state_mode(ad2_ctx ctx, int32_t mode);

/* Cost of the variant-2 iteration kernel (C_ij = ||x_i - y_j||^2, recomputed every
 * iteration from the staged supports):
 *   1 (the environment variable AD2_TC=1 makes it the default): for fp32 rounds whose passes are single
 *     32-row members (m <= 32, m_k <= 32, 32 row blocks) with 4 < d <= 16, the dot products
 *     x'_i . y'_j of the centred coordinates (x' = x - o, y' = y - o, o the cluster's mean centroid
 *     point; C is translation invariant) run on the tensor cores: tcgen05.mma kind::tf32 with tf32
 *     hi / lo splits of both operands (hi.hi + hi.lo + lo.hi) accumulated in fp32 in TMEM, and
 *     C = |x'|^2 + |y'|^2 - 2 x'.y' in fp32.  ad2_info.tc_cost reports whether it is in use.
 *   0 (default): the dot products in fp32 FMAs (packed FFMA2) on the CUDA cores.  Measured on
 *     config 5 the tensor-core form is slower (9.65 vs 8.75 ms per iteration: the per-pass operand
 *     split and six single-thread MMA issues cost what the dot products saved).
 * Takes effect at the next ad2_badmm_step; AD2_ERR_ARG for other values. */
ad2_status ad2_set_tc_cost(ad2_ctx ctx, int32_t enable);

/* Start a round (a1-a3 of SURVEY.md §8(a)): copy/sort the batch by cluster, build C, compute
 * rho per cluster (fixed for the round, X2), Lambda = 0, Pi^(2) = product measure or, for
 * members with warm_mask[k] != 0, the Pi^(2) this context holds for that member from the
 * previous round (its m_k and the ctx m/dtype must be unchanged; else AD2_ERR_ARG).
 *   x0 [K][m][d], w0 [K][m]: initial centroids (same memory space as batch->mem), copied.
 *   warm_mask: host [N] or NULL (all cold).   rho_out: host double[K] or NULL.
 * Synchronises.  Returns AD2_ERR_EMPTY / AD2_ERR_ZERO_RHO per cluster conditions. */
ad2_status ad2_barycenter_init(ad2_ctx ctx, const ad2_batch *batch, const ad2_params *params,
                               const void *x0, const void *w0, const uint8_t *warm_mask,
                               double *rho_out);

/* Host-batch prefetch (pipelining a stream of rounds): enqueue the host->device copies of a host
 * batch (batch->mem == AD2_HOST; offsets, labels, supports, weights) on an internal copy stream,
 * so they overlap whatever the context's stream is running (e.g. the current round).  The next
 * ad2_barycenter_init with the same four host pointers and sizes uses those copies instead of
 * copying again (it waits for them on its stream); any other init discards them.  The host
 * arrays must stay valid and unchanged until that init returns (page-locked memory for an
 * asynchronous copy).  cost_mode tells the layout of `supports` (AD2_COST_TABLE: int32 symbol
 * ids).  Asynchronous; no state change besides the staging buffers. */
ad2_status ad2_prefetch(ad2_ctx ctx, const ad2_batch *batch, ad2_cost_mode cost_mode);

/* n_iters >= 0 B-ADMM iterations at fixed x (a4-a8), then the support-update partial sums of
 * the final Pi^(2) are formed for ad2_update_support.  Asynchronous (one CUDA graph per n). */
ad2_status ad2_badmm_step(ad2_ctx ctx, int32_t n_iters);

/* a9: x update from the Pi^(2) of the last step (Eq.updatex), C rebuilt.  AD2_ERR_STATE if no
 * step has run since init.  Asynchronous. */
ad2_status ad2_update_support(ad2_ctx ctx);

/* a10: obj_out (host double[K]) = (1/N_c) sum_k <C^(k), Pi^(k,1)> with the last Pi^(1) and the
 * current x.  AD2_ERR_STATE if no step has run since init.  Synchronises. */
ad2_status ad2_objective(ad2_ctx ctx, double *obj_out);

/* Cost table for AD2_COST_TABLE rounds: D [V][V] row-major (D[a*V + b] = cost between centroid
 * symbol a and member symbol b, any non-negative values), in `dtype` (must match the batch dtype
 * of the rounds that use it) and `where` memory; copied.  Synchronous. */
ad2_status ad2_set_cost_table(ad2_ctx ctx, const void *D, int32_t V, ad2_dtype dtype, ad2_mem where);

/* Assignment step of AD2-clustering (Alg. 1, reading X13):
 * for every member k of `batch` (the caller's ragged layout, dtype and mem as in init; the
 * batch's labels are ignored) l^(k) = argmin_c W_2^2(P_c, P^(k)), the exact optimal-transport
 * cost (Eq.primal, squared Euclidean ground cost) to each centroid c of
 * (x [K][m][d], w [K][m]) in batch->dtype and batch->mem; ties go to the lowest c.  Weights of
 * both sides are renormalised in fp64; the whole step runs in fp64 on the device (mean and
 * relaxed-marginal lower bounds prune centroids, survivors are solved exactly by successive
 * shortest paths).  Outputs in `where` memory: labels_out [N] (int32), w2_out [N] (double, the
 * minimum W_2^2; may be NULL).  n_exact_out (host, may be NULL): exact problems solved.
 * Synchronous.  Independent of the B-ADMM round state (needs only a created context).
 * Errors: AD2_ERR_ARG for bad shapes / offsets / a member + centroid pair whose workspace does
 * not fit in shared memory; AD2_ERR_NONFINITE if a transport solve failed to terminate. */
ad2_status ad2_assign(ad2_ctx ctx, const ad2_batch *batch, const void *x, const void *w,
                      int32_t *labels_out, double *w2_out, ad2_mem where, int64_t *n_exact_out);
/* The same for symbolic supports: batch->d = 1 with int32 symbol ids in supports,
 * xs [K][m] int32 centroid symbols, cost from the context's table (ad2_set_cost_table, batch
 * dtype); there is no mean bound (centroids visited in index order, relaxed-marginal bounds
 * prune).  AD2_ERR_ARG for an id outside [0, V). */
ad2_status ad2_assign_symbolic(ad2_ctx ctx, const ad2_batch *batch, const int32_t *xs, const void *w,
                               int32_t *labels_out, double *w2_out, ad2_mem where, int64_t *n_exact_out);

/* Current centroids: x [K][m][d], w [K][m] in the ctx dtype, into `where` memory. */
ad2_status ad2_get_centroids(ad2_ctx ctx, void *x, void *w, ad2_mem where);

/* One state array for all members of this rank, in the caller's ORIGINAL member order:
 * member k's m x m_k block at out + m*offsets[k], COLUMN-major (entry (i,j) at j*m + i).
 * `which` selects Pi^(1), Pi^(2), Lambda or the cost C.  Synchronises for AD2_HOST. */
ad2_status ad2_get_plans(ad2_ctx ctx, int which, void *out, ad2_mem where);

/* Per-cluster rho (host double[K]) of the current round. */
ad2_status ad2_get_rho(ad2_ctx ctx, double *rho_out);

ad2_status ad2_get_info(ad2_ctx ctx, ad2_info *info);

/* Kernel timing: enable = 1 brackets every B-ADMM iteration-kernel launch of later steps by CUDA
 * events on the launching stream (event-record nodes inside the step graph); enable = 2 does so
 * for the next ad2_badmm_step call only (later steps run the plain graph: no timing overhead);
 * 0 turns it off.  Other values: AD2_ERR_ARG.  ad2_prof_read fills
 * launch_ms[0..min(capacity, n)-1] with the durations (ms) of the most recent profiled step's
 * launches in order [first (phase 1 only), fused x (n_iters-1), last (phase 2 only)],
 * *n_launches = n_iters + 1 (n_iters when the last pass also forms the support-update partials:
 * the variant-2 kernel and n_iters >= 2), and *step_ms = first start to last end.  Synchronises. */
ad2_status ad2_set_profiling(ad2_ctx ctx, int enable);
ad2_status ad2_prof_read(ad2_ctx ctx, double *launch_ms, int64_t capacity, int64_t *n_launches,
                         double *step_ms);

/* Centroid initialisation (§V, Eq.merge; part of SURVEY.md §8(f) NEXT #2):
 * for every cluster c the caller picks a member pick[c] (host int64 [K], index into the batch;
 * the paper picks one at random among the cluster's members with at least m support points), and
 * its support (weights renormalised in fp64) is reduced to m points by repeatedly merging the pair
 * minimising w_i w_j |x_i - x_j|^2 / (w_i + w_j) into its weighted mean (ties: lowest (i, j));
 * a member with fewer than m points has its heaviest point split in halves (reading X19).
 * Runs in fp64 on the device; x0_out [K][m][d], w0_out [K][m] (batch dtype) in `where` memory.
 * batch->K, m, d give the shapes; its labels are ignored.  Synchronous. */
ad2_status ad2_merge_init(ad2_ctx ctx, const ad2_batch *batch, const int64_t *pick, void *x0_out, void *w0_out,
                          ad2_mem where);

/* Initial partition.  Alg. 1 starts from "K random centroid[s]"
 * and a labelling; the recipe is k-means++ on member means (the paper's own
 * comparison method), every member labelled to its nearest mean, then per cluster a
 * random member with >= m support points reduced by Eq.merge (ad2_merge_init).
 * Every random draw is an argument; X20-X23 fix how a draw becomes an index.  All
 * arithmetic is fp64 with fixed summation orders (ad2_seed.cu); synchronous; single-rank calls
 * (a sharded job runs the seeding once and broadcasts the K*d centres).  Host batches are staged
 * in the context's staging buffers, as for ad2_merge_init.
 *
 * ad2_kmeanspp: member means mean(P^(k)) = sum_j w_j y_j of the members sample[0..ns) (host int64,
 * each in [0, N)), k-means++ D^2 seeding with the uniforms u[0..K) (host, each in [0, 1)): centre 0
 * = sampled mean floor(u_0 ns), centre c = the first sampled mean whose prefix sum of D^2 exceeds
 * u_c * sum D^2 (X20), then lloyd_iters Lloyd iterations (X21).  batch->K, d give the shapes
 * (1 <= d <= 256, ns >= K); labels and m are ignored.  centres_out [K][d] fp64 in `where` memory.
 * AD2_ERR_ARG on a bad shape, sample index or uniform. */
ad2_status ad2_kmeanspp(ad2_ctx ctx, const ad2_batch *batch, const int64_t *sample, int64_t ns, const double *u,
                        int32_t lloyd_iters, double *centres_out, ad2_mem where);
/* ad2_label_nearest: every member's mean to its nearest centre (ties: lowest index, X21), then while
 * a cluster is empty the lowest empty cluster takes the member farthest from its own centre among
 * clusters with >= 2 members (lowest index on ties) and that member's mean becomes its centre
 * (X22).  centres [K][d] fp64 in `where` memory (read), labels_out [N] int32 and centres_out
 * [K][d] fp64 (the centres after the repair) in `where` memory.  Needs N >= K. */
ad2_status ad2_label_nearest(ad2_ctx ctx, const ad2_batch *batch, const double *centres, int32_t *labels_out,
                             double *centres_out, ad2_mem where);
/* ad2_pick_members: per cluster c the member whose support initialises the centroid (X23): among
 * c's members with m_k >= batch->m in index order the one at position floor(u_c * n_big) (u host
 * double [K] in [0, 1)), else the first member of c with the largest m_k.  Needs batch->labels.
 * pick_out host int64 [K] (feed it to ad2_merge_init).  AD2_ERR_EMPTY if a cluster has no member. */
ad2_status ad2_pick_members(ad2_ctx ctx, const ad2_batch *batch, const double *u, int64_t *pick_out);

/* The AD2 outer loop (Alg. 1, P:259-266 with Alg. 4 as the centroid update; SURVEY.md §8(f)
 * NEXT #2), on the device: the shard is staged once and stays on this GPU; each
 * round r = ad2_barycenter_init (round 0 cold; later rounds warm-start Pi^(2) for members whose
 * label did not change; Lambda reset, X7) -> T iterations with a support update every
 * tau (X6) -> [ad2_objective into obj_out[r*K..]] -> ad2_assign against the new centroids.
 * Stops after max_rounds or when the fraction of members (all ranks) whose label changed is
 * <= stop_frac.  batch->labels are the initial labels; x0/w0 the initial centroids (batch->mem).
 * Outputs: labels_out [N] (batch->mem; the last assignment), rounds_out (host), changed_out
 * [max_rounds] (host, may be NULL), obj_out [max_rounds*K] (host, may be NULL).  On return the
 * context holds the last round (ad2_get_centroids gives the centroids the labels refer to).
 * AD2_ERR_EMPTY (labels_out still written) if an assignment leaves a cluster without members. */
typedef struct {
    int32_t T;                  /* B-ADMM iterations per round */
    int32_t tau;                /* support update every tau iterations */
    int32_t max_rounds;         /* outer iterations, >= 1 */
    double stop_frac;           /* stop when changed labels / N <= stop_frac (0: only when stable) */
} ad2_loop;

ad2_status ad2_cluster(ad2_ctx ctx, const ad2_batch *batch, const ad2_params *params, const ad2_loop *loop,
                       const void *x0, const void *w0, int32_t *labels_out, int32_t *rounds_out,
                       double *changed_out, double *obj_out);

/* Wait for all work of the context; returns a latched device error if any. */
ad2_status ad2_sync(ad2_ctx ctx);

const char *ad2_last_error(ad2_ctx ctx);
const char *ad2_status_string(ad2_status s);
void ad2_destroy(ad2_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* AD2_H */
