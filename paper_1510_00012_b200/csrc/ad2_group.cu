// ad2_group.cu — a host-memory process group for libad2's cross-rank sums (include/ad2.h,
// "Host process group").  Host code only.
//
// The multi-GPU path all-reduces per-cluster partial sums with NCCL (the paper's
// per-iteration synchronisation).  NCCL needs one GPU per rank, so the
// sharded path could never run with more than one rank on a one-GPU box.  This group replaces
// the transport, not the algorithm: ranks are processes on one host that share a POSIX
// shared-memory segment; an all-reduce copies this rank's buffer into its slot, waits at a
// barrier, sums the slots in rank order 0..n-1 (so every rank gets the bit-identical result),
// and waits at a second barrier before any slot is reused.  Inside libad2 a collective becomes
// a device->host copy, a host-function node running this all-reduce, and a host->device copy,
// all capturable in the step's CUDA graph.  No kernel ever waits on another rank.
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "../../include/ad2.h"
#include "ad2_group.h"

namespace {
struct alignas(64) Header {
  std::atomic<int32_t> joined;     // ranks that mapped the segment
  std::atomic<int32_t> arrive;     // barrier arrivals
  std::atomic<int32_t> sense;      // barrier generation (sense-reversing)
  int32_t nranks;
  int64_t slot_bytes;
};
constexpr size_t HDR = 256;

double now_s() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}
}  // namespace

struct ad2_group_s {
  int nranks = 1, rank = 0;
  size_t slot = 0, map_bytes = 0;
  char* base = nullptr;
  int32_t local_sense = 0;
  double timeout_s = 300.0;
  std::atomic<int> failed{0};          // a barrier timed out: every later collective is void
  Header* hdr() const { return reinterpret_cast<Header*>(base); }
  char* slot_ptr(int r) const { return base + HDR + (size_t)r * slot; }
  bool barrier() {
    if (failed.load()) return false;
    local_sense ^= 1;
    Header* h = hdr();
    if (h->arrive.fetch_add(1, std::memory_order_acq_rel) == nranks - 1) {
      h->arrive.store(0, std::memory_order_relaxed);
      h->sense.store(local_sense, std::memory_order_release);
      return true;
    }
    const double t0 = now_s();
    int spins = 0;
    while (h->sense.load(std::memory_order_acquire) != local_sense) {
      if (++spins > 256) {
        sched_yield();
        if ((spins & 1023) == 0 && now_s() - t0 > timeout_s) {
          failed.store(1);
          return false;
        }
      }
    }
    return true;
  }
};

template <typename T>
static void sum_slots(ad2_group g, void* out, size_t count) {
  T* o = static_cast<T*>(out);
  const T* s0 = reinterpret_cast<const T*>(g->slot_ptr(0));
  for (size_t i = 0; i < count; ++i) o[i] = s0[i];
  for (int r = 1; r < g->nranks; ++r) {
    const T* sr = reinterpret_cast<const T*>(g->slot_ptr(r));
    for (size_t i = 0; i < count; ++i) o[i] += sr[i];
  }
}

size_t ad2_group_type_size(int dtype) {
  switch (dtype) {
    case AD2_GROUP_F32: return 4;
    case AD2_GROUP_F64: return 8;
    case AD2_GROUP_U64: return 8;
  }
  return 0;
}

int ad2_group_sum_host(ad2_group g, void* buf, size_t count, int dtype) {
  const size_t es = ad2_group_type_size(dtype);
  if (!g || !buf || !es) return 1;
  if (count * es > g->slot) {
    g->failed.store(1);
    return 2;
  }
  if (g->nranks == 1) return g->failed.load() ? 3 : 0;
  memcpy(g->slot_ptr(g->rank), buf, count * es);
  if (!g->barrier()) return 3;
  if (dtype == AD2_GROUP_F32) sum_slots<float>(g, buf, count);
  else if (dtype == AD2_GROUP_F64) sum_slots<double>(g, buf, count);
  else sum_slots<unsigned long long>(g, buf, count);
  if (!g->barrier()) return 3;
  return 0;
}

bool ad2_group_failed(ad2_group g) { return g && g->failed.load() != 0; }
int ad2_group_rank(ad2_group g) { return g ? g->rank : 0; }
int ad2_group_size(ad2_group g) { return g ? g->nranks : 1; }

ad2_status ad2_group_open(ad2_group* out, const char* name, int nranks, int rank, int64_t slot_bytes) {
  if (!out) return AD2_ERR_ARG;
  *out = nullptr;
  if (!name || name[0] != '/' || nranks < 1 || rank < 0 || rank >= nranks || slot_bytes < 64) return AD2_ERR_ARG;
  ad2_group g = new (std::nothrow) ad2_group_s();
  if (!g) return AD2_ERR_OOM;
  g->nranks = nranks;
  g->rank = rank;
  g->slot = ((size_t)slot_bytes + 63) / 64 * 64;
  g->map_bytes = HDR + (size_t)nranks * g->slot;
  if (const char* t = getenv("AD2_GROUP_TIMEOUT")) g->timeout_s = atof(t);
  // every rank creates-or-opens and sizes the segment (ftruncate to the same size is idempotent;
  // a fresh segment reads as zeros, which is the header's initial state)
  int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
  if (fd < 0 || ftruncate(fd, (off_t)g->map_bytes) != 0) {
    if (fd >= 0) close(fd);
    delete g;
    return AD2_ERR_ARG;
  }
  void* p = mmap(nullptr, g->map_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    delete g;
    return AD2_ERR_OOM;
  }
  g->base = static_cast<char*>(p);
  Header* h = g->hdr();
  h->joined.fetch_add(1);
  const double t0 = now_s();
  while (h->joined.load() < nranks) {        // every rank has mapped the segment
    sched_yield();
    if (now_s() - t0 > g->timeout_s) {
      munmap(g->base, g->map_bytes);
      delete g;
      return AD2_ERR_STATE;
    }
  }
  if (!g->barrier()) {
    munmap(g->base, g->map_bytes);
    delete g;
    return AD2_ERR_STATE;
  }
  if (rank == 0) shm_unlink(name);           // the mappings keep the segment alive
  *out = g;
  return AD2_OK;
}

ad2_status ad2_group_allreduce(ad2_group g, void* host_buf, int64_t count, int32_t dtype) {
  if (!g || !host_buf || count < 0) return AD2_ERR_ARG;
  const int r = ad2_group_sum_host(g, host_buf, (size_t)count, dtype);
  return r == 0 ? AD2_OK : (r == 3 ? AD2_ERR_NCCL : AD2_ERR_ARG);
}

void ad2_group_close(ad2_group g) {
  if (!g) return;
  if (g->base) munmap(g->base, g->map_bytes);
  delete g;
}
