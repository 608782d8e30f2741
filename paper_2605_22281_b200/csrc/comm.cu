// Collectives for the sharded path: NCCL (dlopen) and the in-process LocalGroup.
#include "comm.h"

#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <vector>

namespace sfl {

// CUDA IPC exchange of one cudaMalloc'ed buffer per rank (the peer-memory collectives of the
// process transports): `gather` is the transport's blocking host all-gather.
template <class Gather>
static int ipc_share(int rank, int world, void* local, void** peers, Gather gather, std::string& err) {
  cudaIpcMemHandle_t mine;
  if (cudaIpcGetMemHandle(&mine, local) != cudaSuccess) {
    cudaGetLastError();
    err = "cudaIpcGetMemHandle failed";
    return -1;
  }
  std::vector<cudaIpcMemHandle_t> all(world);
  if (gather(&mine, all.data(), sizeof(mine))) return -1;
  for (int r = 0; r < world; ++r) {
    peers[r] = nullptr;
    if (r == rank) {
      peers[r] = local;
    } else if (cudaIpcOpenMemHandle(&peers[r], all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      err = "cudaIpcOpenMemHandle failed (no peer access between the ranks' GPUs?)";
      for (int q = 0; q < r; ++q)
        if (q != rank && peers[q]) cudaIpcCloseMemHandle(peers[q]);
      return -1;
    }
  }
  return 0;
}

// ====================================================================== NCCL
namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, []() {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // e.g. PyTorch's, already loaded
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
#define SFL_SYM(field, name)                                        \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(lib, name)); \
  if (!api.field) {                                                 \
    api.why = std::string("missing NCCL symbol ") + name;           \
    return;                                                         \
  }
    SFL_SYM(GetUniqueId, "ncclGetUniqueId");
    SFL_SYM(CommInitRank, "ncclCommInitRank");
    SFL_SYM(CommDestroy, "ncclCommDestroy");
    SFL_SYM(AllReduce, "ncclAllReduce");
    SFL_SYM(AllGather, "ncclAllGather");
    SFL_SYM(ReduceScatter, "ncclReduceScatter");
    SFL_SYM(GetErrorString, "ncclGetErrorString");
#undef SFL_SYM
    api.ok = true;
  });
  return api;
}

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  double* scratch = nullptr;  // one double for the barrier all-reduce
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
    cudaFree(scratch);
  }
  int barrier(cudaStream_t s, std::string& err) override {
    if (!scratch && cudaMalloc(&scratch, sizeof(double)) != cudaSuccess) {
      err = "barrier: cudaMalloc failed";
      return -1;
    }
    // an all-reduce completes only after every rank's NCCL kernel ran, i.e. after all the work its
    // stream had before it (the kernels storing into peer memory)
    return check(nccl().AllReduce(scratch, scratch, 1, ncclDouble, ncclSum, comm, s), "ncclAllReduce(barrier)", err);
  }
  int share_buffer(void* local, void** peers, std::string& err) override {
    return ipc_share(rank, world, local, peers,
                     [&](const void* a, void* b, size_t n) { return allgather_host(a, b, n, err); }, err);
  }
  void unshare_buffer(void** peers) override {
    for (int r = 0; r < world; ++r)
      if (r != rank && peers[r]) cudaIpcCloseMemHandle(peers[r]);
  }
  void release_fence() override {
    std::string e;
    if (!barrier(nullptr, e)) cudaStreamSynchronize(nullptr);
  }
  int check(ncclResult_t r, const char* what, std::string& err) {
    if (r == ncclSuccess) return 0;
    err = std::string(what) + ": " + nccl().GetErrorString(r);
    return -1;
  }
  int allreduce(double* buf, size_t count, bool is_max, cudaStream_t s, std::string& err) override {
    return check(nccl().AllReduce(buf, buf, count, ncclDouble, is_max ? ncclMax : ncclSum, comm, s), "ncclAllReduce",
                 err);
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) override {
    return check(nccl().AllGather(send, recv, count, ncclDouble, comm, s), "ncclAllGather", err);
  }
  int reduce_scatter(const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) override {
    return check(nccl().ReduceScatter(send, recv, count, ncclDouble, ncclSum, comm, s), "ncclReduceScatter", err);
  }
  int allgather_host(const void* send, void* recv, size_t bytes, std::string& err) override {
    void *ds = nullptr, *dr = nullptr;
    if (cudaMalloc(&ds, bytes) != cudaSuccess || cudaMalloc(&dr, bytes * world) != cudaSuccess) {
      cudaFree(ds);
      err = "allgather_host: cudaMalloc failed";
      return -1;
    }
    cudaMemcpy(ds, send, bytes, cudaMemcpyHostToDevice);
    int rc = check(nccl().AllGather(ds, dr, bytes, ncclChar, comm, 0), "ncclAllGather(host)", err);
    if (!rc) {
      cudaStreamSynchronize(0);
      cudaMemcpy(recv, dr, bytes * world, cudaMemcpyDeviceToHost);
    }
    cudaFree(ds);
    cudaFree(dr);
    return rc;
  }
};

}  // namespace

int nccl_get_unique_id(uint8_t id[128], std::string& err) {
  NcclApi& a = nccl();
  if (!a.ok) {
    err = a.why;
    return -1;
  }
  ncclUniqueId u;
  ncclResult_t r = a.GetUniqueId(&u);
  if (r != ncclSuccess) {
    err = std::string("ncclGetUniqueId: ") + a.GetErrorString(r);
    return -1;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return 0;
}

Comm* nccl_comm_create(const uint8_t id[128], int rank, int world, int device, std::string& err) {
  NcclApi& a = nccl();
  if (!a.ok) {
    err = a.why;
    return nullptr;
  }
  cudaSetDevice(device);
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  NcclComm* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  ncclResult_t r = a.CommInitRank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + a.GetErrorString(r);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

// ====================================================================== in-process group
constexpr int kMaxLocal = 8;

struct PtrSet {
  const double* in[kMaxLocal];
  double* out[kMaxLocal];
};

__global__ void k_local_allreduce(PtrSet p, int world, size_t count, int is_max) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double acc = p.in[0][i];
    for (int r = 1; r < world; ++r) acc = is_max ? fmax(acc, p.in[r][i]) : acc + p.in[r][i];
    for (int r = 0; r < world; ++r) p.out[r][i] = acc;
  }
}
__global__ void k_local_allgather(PtrSet p, int world, size_t count) {
  const size_t total = count * world;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)(i / count);
    const double v = p.in[q][i - q * count];
    for (int r = 0; r < world; ++r) p.out[r][i] = v;
  }
}
__global__ void k_local_reduce_scatter(PtrSet p, int world, size_t count) {
  const size_t total = count * world;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / count);
    double acc = p.in[0][i];
    for (int q = 1; q < world; ++q) acc += p.in[q][i];
    p.out[r][i - r * count] = acc;
  }
}

struct LocalGroup {
  int world = 1, device = 0;
  std::mutex mu;
  std::condition_variable cv;
  int refs = 0;
  int arrived = 0, left = 0;
  uint64_t gen = 0, gen2 = 0;
  cudaStream_t cs = nullptr;
  cudaEvent_t done = nullptr;
  cudaEvent_t ev[kMaxLocal];
  const void* send[kMaxLocal];
  void* recv[kMaxLocal];
  std::vector<char> host_stage;
  int status = 0;
};

namespace {

struct LocalComm : Comm {
  LocalGroup* g = nullptr;

  // kind: 0 allreduce-sum, 1 allreduce-max, 2 allgather, 3 reduce-scatter, 4 host allgather
  int collective(int kind, const void* send, void* recv, size_t count, cudaStream_t s, std::string& err) {
    LocalGroup& G = *g;
    if (kind != 4) cudaEventRecord(G.ev[rank], s);
    std::unique_lock<std::mutex> lk(G.mu);
    G.send[rank] = send;
    G.recv[rank] = recv;
    if (kind == 4) std::memcpy(G.host_stage.data() + rank * count, send, count);
    const uint64_t my = G.gen;
    if (++G.arrived == G.world) {
      G.status = 0;
      if (kind != 4) {
        for (int r = 0; r < G.world; ++r) cudaStreamWaitEvent(G.cs, G.ev[r], 0);
        PtrSet p;
        for (int r = 0; r < G.world; ++r) {
          p.in[r] = static_cast<const double*>(G.send[r]);
          p.out[r] = static_cast<double*>(G.recv[r]);
        }
        const size_t total = (kind >= 2) ? count * G.world : count;
        const int grid = (int)std::min<size_t>((total + 255) / 256, 148 * 4);
        if (grid > 0) {
          if (kind <= 1)
            k_local_allreduce<<<grid, 256, 0, G.cs>>>(p, G.world, count, kind == 1);
          else if (kind == 2)
            k_local_allgather<<<grid, 256, 0, G.cs>>>(p, G.world, count);
          else
            k_local_reduce_scatter<<<grid, 256, 0, G.cs>>>(p, G.world, count);
        }
        if (cudaGetLastError() != cudaSuccess) G.status = -1;
        cudaEventRecord(G.done, G.cs);
      }
      G.arrived = 0;
      ++G.gen;
      G.cv.notify_all();
    } else {
      G.cv.wait(lk, [&] { return G.gen != my; });
    }
    const int st = G.status;
    if (kind == 4) std::memcpy(recv, G.host_stage.data(), count * G.world);
    lk.unlock();
    if (kind != 4) cudaStreamWaitEvent(s, G.done, 0);
    // second rendezvous: nobody re-records `done` before every rank has waited on it
    lk.lock();
    const uint64_t my2 = G.gen2;
    if (++G.left == G.world) {
      G.left = 0;
      ++G.gen2;
      G.cv.notify_all();
    } else {
      G.cv.wait(lk, [&] { return G.gen2 != my2; });
    }
    if (st) err = "local collective kernel launch failed";
    return st;
  }

  int allreduce(double* buf, size_t count, bool is_max, cudaStream_t s, std::string& err) override {
    return collective(is_max ? 1 : 0, buf, buf, count, s, err);
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) override {
    return collective(2, send, recv, count, s, err);
  }
  int reduce_scatter(const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) override {
    return collective(3, send, recv, count, s, err);
  }
  int allgather_host(const void* send, void* recv, size_t bytes, std::string& err) override {
    {
      std::lock_guard<std::mutex> lk(g->mu);
      if (g->host_stage.size() < bytes * g->world) g->host_stage.resize(bytes * g->world);
    }
    return collective(4, send, recv, bytes, nullptr, err);
  }
  // every rank's stream waits on every rank's prior work (a zero-length collective: no kernel)
  int barrier(cudaStream_t s, std::string& err) override { return collective(0, nullptr, nullptr, 0, s, err); }
  int share_buffer(void* local, void** peers, std::string& err) override {
    return allgather_host(&local, peers, sizeof(void*), err);
  }
  ~LocalComm() override { local_group_release(g); }
};

}  // namespace

LocalGroup* local_group_create(int world, int device, std::string& err) {
  if (world < 1 || world > kMaxLocal) {
    err = "local group size must be 1..8";
    return nullptr;
  }
  cudaSetDevice(device);
  LocalGroup* g = new LocalGroup();
  g->world = world;
  g->device = device;
  g->refs = 1;
  g->host_stage.resize(4096);
  if (cudaStreamCreateWithFlags(&g->cs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming) != cudaSuccess) {
    err = "local group: stream/event creation failed";
    delete g;
    return nullptr;
  }
  for (int r = 0; r < world; ++r) cudaEventCreateWithFlags(&g->ev[r], cudaEventDisableTiming);
  return g;
}

void local_group_release(LocalGroup* g) {
  if (!g) return;
  bool last;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    last = --g->refs == 0;
  }
  if (last) {
    cudaSetDevice(g->device);
    cudaStreamSynchronize(g->cs);
    for (int r = 0; r < g->world; ++r) cudaEventDestroy(g->ev[r]);
    cudaEventDestroy(g->done);
    cudaStreamDestroy(g->cs);
    delete g;
  }
}

Comm* local_comm_create(LocalGroup* g, int rank) {
  if (!g || rank < 0 || rank >= g->world) return nullptr;
  {
    std::lock_guard<std::mutex> lk(g->mu);
    g->refs++;
  }
  LocalComm* c = new LocalComm();
  c->g = g;
  c->rank = rank;
  c->world = g->world;
  return c;
}


// ====================================================================== processes + CUDA IPC
// World processes of one node (one GPU each, or several on one GPU): host rendezvous through a
// POSIX shared-memory segment, data through CUDA-IPC peer memory.  Every collective stages its
// input in a per-rank device buffer the peers opened with cudaIpcOpenMemHandle, meets the other
// ranks on the host after a stream synchronise, and reduces the peers' buffers in fixed rank order
// with one kernel (the same order as the in-process group: identical bits).  No kernel waits on
// another rank.  A peer that never arrives fails the call after kIpcTimeoutS instead of hanging.
namespace {

constexpr int kIpcTimeoutS = 180;
constexpr size_t kIpcStage = 4096;

struct ShmHdr {
  std::atomic<int> arrived;
  std::atomic<unsigned> gen;
  char stage[kMaxLocal][kIpcStage];
};

__global__ void k_ipc_allreduce(PtrSet p, int world, size_t count, int is_max, double* out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double acc = p.in[0][i];
    for (int r = 1; r < world; ++r) acc = is_max ? fmax(acc, p.in[r][i]) : acc + p.in[r][i];
    out[i] = acc;
  }
}
__global__ void k_ipc_allgather(PtrSet p, int world, size_t count, double* out) {
  const size_t total = count * world;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)(i / count);
    out[i] = p.in[q][i - q * count];
  }
}
__global__ void k_ipc_reduce_scatter(PtrSet p, int world, size_t count, int rank, double* out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double acc = p.in[0][rank * count + i];
    for (int q = 1; q < world; ++q) acc += p.in[q][rank * count + i];
    out[i] = acc;
  }
}

struct IpcComm : Comm {
  ShmHdr* shm = nullptr;
  std::string name;
  double* stg = nullptr;  // this rank's staging buffer (peers read it)
  size_t cap = 0;         // bytes
  void* peers[kMaxLocal] = {};

  ~IpcComm() override {
    if (stg) {
      std::string e;
      host_barrier(e);  // nobody still reads a peer's staging buffer
      unshare_buffer(peers);
      host_barrier(e);
      cudaFree(stg);
    }
    if (shm) munmap(shm, sizeof(ShmHdr));
  }
  int host_barrier(std::string& err) {
    const unsigned my = shm->gen.load(std::memory_order_acquire);
    if (shm->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == world) {
      shm->arrived.store(0, std::memory_order_relaxed);
      shm->gen.fetch_add(1, std::memory_order_release);
      return 0;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned spin = 0; shm->gen.load(std::memory_order_acquire) == my; ++spin) {
      if ((spin & 1023) == 1023) {
        sched_yield();
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(kIpcTimeoutS)) {
          err = "ipc communicator: a rank did not reach the rendezvous within the timeout";
          return -1;
        }
      }
    }
    return 0;
  }
  int allgather_host(const void* send, void* recv, size_t bytes, std::string& err) override {
    if (bytes > kIpcStage) {
      err = "ipc communicator: host all-gather larger than its stage";
      return -1;
    }
    std::memcpy(shm->stage[rank], send, bytes);
    if (host_barrier(err)) return -1;
    for (int r = 0; r < world; ++r) std::memcpy(static_cast<char*>(recv) + r * bytes, shm->stage[r], bytes);
    return host_barrier(err);
  }
  int share_buffer(void* local, void** out, std::string& err) override {
    return ipc_share(rank, world, local, out,
                     [&](const void* a, void* b, size_t n) { return allgather_host(a, b, n, err); }, err);
  }
  void unshare_buffer(void** ps) override {
    for (int r = 0; r < world; ++r)
      if (r != rank && ps[r]) cudaIpcCloseMemHandle(ps[r]);
  }
  void release_fence() override {
    std::string e;
    host_barrier(e);
  }
  // every rank calls every collective with the same count, so the staging buffers grow together
  int ensure(size_t bytes, std::string& err) {
    if (bytes <= cap) return 0;
    if (stg) {
      if (host_barrier(err)) return -1;
      unshare_buffer(peers);
      if (host_barrier(err)) return -1;
      cudaFree(stg);
      stg = nullptr;
      cap = 0;
    }
    const size_t want = std::max<size_t>(bytes + bytes / 2, (size_t)2 << 20);  // its own driver block
    if (cudaMalloc(&stg, want) != cudaSuccess) {
      cudaGetLastError();
      err = "ipc communicator: staging cudaMalloc failed";
      return -1;
    }
    if (share_buffer(stg, peers, err)) return -1;
    cap = want;
    return 0;
  }
  // kind: 0 sum, 1 max, 2 all-gather, 3 reduce-scatter
  int collective(int kind, const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) {
    const size_t in_count = kind == 3 ? count * world : count;
    if (ensure(in_count * sizeof(double), err)) return -1;
    if (in_count) cudaMemcpyAsync(stg, send, in_count * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) {
      err = "ipc communicator: stream failed before a collective";
      return -1;
    }
    if (host_barrier(err)) return -1;  // every rank's input is staged
    if (in_count) {
      PtrSet p;
      for (int r = 0; r < world; ++r) {
        p.in[r] = static_cast<const double*>(peers[r]);
        p.out[r] = nullptr;
      }
      const size_t total = kind == 2 ? count * world : count;
      const int grid = (int)std::min<size_t>((total + 255) / 256, 148 * 4);
      if (kind <= 1)
        k_ipc_allreduce<<<grid, 256, 0, s>>>(p, world, count, kind == 1, recv);
      else if (kind == 2)
        k_ipc_allgather<<<grid, 256, 0, s>>>(p, world, count, recv);
      else
        k_ipc_reduce_scatter<<<grid, 256, 0, s>>>(p, world, count, rank, recv);
      if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) {
        err = "ipc communicator: collective kernel failed";
        return -1;
      }
    }
    return host_barrier(err);  // every rank has read every staging buffer
  }
  int allreduce(double* buf, size_t count, bool is_max, cudaStream_t s, std::string& err) override {
    return collective(is_max ? 1 : 0, buf, buf, count, s, err);
  }
  int allgather(const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) override {
    return collective(2, send, recv, count, s, err);
  }
  int reduce_scatter(const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) override {
    return collective(3, send, recv, count, s, err);
  }
  int barrier(cudaStream_t s, std::string& err) override {
    if (cudaStreamSynchronize(s) != cudaSuccess) {
      err = "ipc communicator: stream failed before a barrier";
      return -1;
    }
    return host_barrier(err);
  }
};

}  // namespace

Comm* ipc_comm_create(const char* shm_name, int rank, int world, int device, std::string& err) {
  if (world < 1 || world > kMaxLocal || !shm_name || shm_name[0] != '/' || std::strlen(shm_name) > 100) {
    err = "ipc communicator: world must be 1..8 and the name a POSIX shm name ('/...', <= 100 chars)";
    return nullptr;
  }
  cudaSetDevice(device);
  // every rank creates-or-opens the segment; a new segment is zero-filled, which is the initial state
  const int fd = shm_open(shm_name, O_CREAT | O_RDWR, 0600);
  if (fd < 0 || ftruncate(fd, sizeof(ShmHdr)) != 0) {
    if (fd >= 0) close(fd);
    err = "ipc communicator: shm_open / ftruncate failed";
    return nullptr;
  }
  void* m = mmap(nullptr, sizeof(ShmHdr), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (m == MAP_FAILED) {
    err = "ipc communicator: mmap failed";
    return nullptr;
  }
  IpcComm* c = new IpcComm();
  c->rank = rank;
  c->world = world;
  c->name = shm_name;
  c->shm = static_cast<ShmHdr*>(m);
  // all ranks have mapped the segment after this rendezvous: the name can go
  const int brc = c->host_barrier(err);
  if (rank == 0) shm_unlink(shm_name);  // also when a rank never came: no stale segment
  if (brc) {
    munmap(c->shm, sizeof(ShmHdr));
    c->shm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}


// ====================================================================== NCCL self-test (one rank)
// Drives every NcclComm entry the sharded path uses through a world-1 communicator: the dlopen'ed
// symbols and their argument order, the host all-gather, the barrier, and the capture of the NCCL
// calls into a CUDA graph with two replays on changed inputs.  A one-rank all-reduce / all-gather /
// reduce-scatter is the identity, so every result is checked against its input.
namespace {
__global__ void k_selftest_fill(double* a, size_t n, double scale) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    a[i] = scale * (double)(i + 1);
}
}  // namespace

int nccl_selftest(int device, std::string& err) {
  uint8_t id[128];
  if (nccl_get_unique_id(id, err)) return -2;
  Comm* c = nccl_comm_create(id, 0, 1, device, err);
  if (!c) return -2;
  const size_t n = 5000;
  double *a = nullptr, *r = nullptr;
  cudaStream_t s = nullptr;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  std::vector<double> ha(n), hr(n);
  int rc = -1;
  auto same = [&](const double* dev, double scale, const char* what) {
    cudaStreamSynchronize(s);
    cudaMemcpy(hr.data(), dev, n * sizeof(double), cudaMemcpyDeviceToHost);
    for (size_t i = 0; i < n; ++i)
      if (hr[i] != scale * (double)(i + 1)) {
        err = std::string("nccl self-test: wrong result after ") + what;
        return false;
      }
    return true;
  };
  do {
    if (cudaMalloc(&a, n * sizeof(double)) != cudaSuccess || cudaMalloc(&r, n * sizeof(double)) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
      err = "nccl self-test: allocation failed";
      break;
    }
    k_selftest_fill<<<8, 256, 0, s>>>(a, n, 1.0);
    if (c->allreduce(a, n, false, s, err) || !same(a, 1.0, "allreduce(sum)")) break;
    if (c->allreduce(a, n, true, s, err) || !same(a, 1.0, "allreduce(max)")) break;
    cudaMemsetAsync(r, 0, n * sizeof(double), s);
    if (c->allgather(a, r, n, s, err) || !same(r, 1.0, "allgather")) break;
    cudaMemsetAsync(r, 0, n * sizeof(double), s);
    if (c->reduce_scatter(a, r, n, s, err) || !same(r, 1.0, "reduce_scatter")) break;
    if (c->barrier(s, err)) break;
    char hs[64], hg[64];
    for (int i = 0; i < 64; ++i) hs[i] = (char)(i * 3 + 1);
    std::memset(hg, 0, sizeof(hg));
    if (c->allgather_host(hs, hg, 64, err)) break;
    if (std::memcmp(hs, hg, 64) != 0) {
      err = "nccl self-test: wrong host all-gather";
      break;
    }
    void* peers[kMaxLocal] = {};
    if (c->share_buffer(a, peers, err)) break;
    if (peers[0] != a) {
      err = "nccl self-test: share_buffer did not return the local buffer for this rank";
      break;
    }
    c->unshare_buffer(peers);
    // the per-iteration graph of the sharded path: kernels and NCCL calls captured together
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      err = "nccl self-test: capture could not start";
      break;
    }
    bool cap_ok = !c->allreduce(a, n, false, s, err) && !c->allgather(a, r, n, s, err) && !c->barrier(s, err);
    if (cudaStreamEndCapture(s, &g) != cudaSuccess || !cap_ok || !g) {
      cudaGetLastError();
      if (err.empty()) err = "nccl self-test: the NCCL calls were not capturable";
      rc = -3;
      break;
    }
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
      err = "nccl self-test: graph instantiation failed";
      rc = -3;
      break;
    }
    bool ok = true;
    for (int rep = 0; rep < 2 && ok; ++rep) {
      const double sc = rep ? -2.5 : 3.0;
      k_selftest_fill<<<8, 256, 0, s>>>(a, n, sc);
      cudaMemsetAsync(r, 0, n * sizeof(double), s);
      ok = cudaGraphLaunch(ge, s) == cudaSuccess && same(r, sc, "graph replay");
      if (!ok && err.empty()) err = "nccl self-test: graph launch failed";
    }
    if (!ok) {
      rc = -3;
      break;
    }
    rc = 0;
  } while (false);
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  if (s) {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  cudaFree(a);
  cudaFree(r);
  delete c;
  cudaGetLastError();
  return rc;
}

}  // namespace sfl
