// Host-staged sum-allreduce between the processes of a world on ONE machine (rs_dist.collective =
// RS_COLL_HOST).  It carries the library's multi-rank code path -- row / column shards, the partial
// sums, the allreduce placement inside the captured iteration graph -- on a machine with fewer GPUs
// than ranks: several rank processes may share one GPU because no kernel ever waits for another
// rank; the wait happens in a host function node of each rank's stream (B200_PROFILING.md: ranks
// that wait on one another in kernels must not share a GPU).  NCCL (RS_COLL_NCCL) is the production
// backend; this one exists so that the world > 1 path is executed and tested.
//
// One allreduce of n doubles = per chunk of at most HC_CHUNK doubles: D2H copy into the rank's
// pinned staging buffer, host function (copy into the rank's slot of a POSIX shared-memory segment,
// barrier, sum of the slots in rank order into staging -- the same sum on every rank --, barrier),
// H2D copy back.  Barriers are generation counters in the segment; a rank that waits more than
// HC_TIMEOUT_S records an error, which rs_solve reports as RS_ENCCL.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "hostcoll.h"

namespace rs {

namespace {

constexpr size_t HC_CHUNK = 1 << 21;   // doubles per staged chunk (16 MB)
constexpr double HC_TIMEOUT_S = 300.0;

struct Shm {
  std::atomic<int> arrive;
  std::atomic<int> gen;
  std::atomic<int> attached;
  int world;
  char pad[128 - 4 * sizeof(int)];
};

}  // namespace

struct HostColl {
  int rank = 0, world = 1;
  std::string name;
  void* base = nullptr;
  size_t map_bytes = 0;
  Shm* hdr = nullptr;
  double* slots = nullptr;     // [world][HC_CHUNK]
  double* staging = nullptr;   // pinned, HC_CHUNK
  std::atomic<int> error{0};
  struct Call {
    HostColl* hc;
    size_t n;
  };
  std::vector<std::unique_ptr<Call>> calls;   // host-node arguments (alive as long as the graphs)

  bool barrier() {
    const int g = hdr->gen.load(std::memory_order_acquire);
    if (hdr->arrive.fetch_add(1, std::memory_order_acq_rel) == world - 1) {
      hdr->arrive.store(0, std::memory_order_relaxed);
      hdr->gen.store(g + 1, std::memory_order_release);
      return true;
    }
    const auto t0 = std::chrono::steady_clock::now();
    int spins = 0;
    while (hdr->gen.load(std::memory_order_acquire) == g) {
      if (++spins > 256) {
        std::this_thread::sleep_for(std::chrono::microseconds(20));
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > HC_TIMEOUT_S)
          return false;
      }
    }
    return true;
  }

  static void CUDART_CB host_fn(void* arg) {
    Call* c = static_cast<Call*>(arg);
    HostColl* h = c->hc;
    if (h->error.load()) return;
    std::memcpy(h->slots + (size_t)h->rank * HC_CHUNK, h->staging, c->n * sizeof(double));
    if (!h->barrier()) {
      h->error.store(1);
      return;
    }
    for (size_t i = 0; i < c->n; ++i) {   // rank order: identical on every rank
      double s = 0.0;
      for (int r = 0; r < h->world; ++r) s += h->slots[(size_t)r * HC_CHUNK + i];
      h->staging[i] = s;
    }
    if (!h->barrier()) h->error.store(1);   // nobody rewrites a slot before all have summed
  }
};

HostColl* hostcoll_create(const char* name, int rank, int world, std::string* err) {
  std::unique_ptr<HostColl> h(new HostColl());
  h->rank = rank;
  h->world = world;
  h->name = name;
  h->map_bytes = sizeof(Shm) + (size_t)world * HC_CHUNK * sizeof(double);
  const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) {
    *err = std::string("shm_open(") + name + "): " + std::strerror(errno);
    return nullptr;
  }
  if (ftruncate(fd, (off_t)h->map_bytes) != 0) {
    *err = std::string("ftruncate: ") + std::strerror(errno);
    close(fd);
    return nullptr;
  }
  h->base = mmap(nullptr, h->map_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (h->base == MAP_FAILED) {
    h->base = nullptr;
    *err = std::string("mmap: ") + std::strerror(errno);
    return nullptr;
  }
  h->hdr = static_cast<Shm*>(h->base);
  h->slots = reinterpret_cast<double*>(static_cast<char*>(h->base) + sizeof(Shm));
  if (cudaMallocHost(&h->staging, HC_CHUNK * sizeof(double)) != cudaSuccess) {
    *err = "cudaMallocHost (host collective staging)";
    return nullptr;
  }
  h->hdr->attached.fetch_add(1);
  if (!h->barrier()) {   // every rank attached before any use
    *err = "host collective: not every rank attached within the timeout";
    return nullptr;
  }
  return h.release();
}

void hostcoll_destroy(HostColl* h) {
  if (!h) return;
  if (h->staging) cudaFreeHost(h->staging);
  if (h->hdr && h->hdr->attached.fetch_sub(1) == 1) shm_unlink(h->name.c_str());
  if (h->base) munmap(h->base, h->map_bytes);
  delete h;
}

bool hostcoll_failed(const HostColl* h) { return h && h->error.load() != 0; }

cudaError_t hostcoll_allreduce(HostColl* h, double* buf, size_t count, cudaStream_t st) {
  for (size_t off = 0; off < count; off += HC_CHUNK) {
    const size_t n = std::min(HC_CHUNK, count - off);
    cudaError_t e = cudaMemcpyAsync(h->staging, buf + off, n * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    h->calls.emplace_back(new HostColl::Call{h, n});
    e = cudaLaunchHostFunc(st, &HostColl::host_fn, h->calls.back().get());
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(buf + off, h->staging, n * sizeof(double), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

void hostcoll_new_name(char* out128) {
  std::random_device rd;
  const unsigned long long a = ((unsigned long long)rd() << 32) ^ rd();
  std::memset(out128, 0, 128);
  std::snprintf(out128, 128, "/rs_hostcoll_%d_%016llx", (int)getpid(), a);
}

}  // namespace rs
