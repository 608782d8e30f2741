// Collectives for the sharded path: NCCL (dlopen) and the in-process LocalGroup.
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <vector>

namespace sfl {

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
    cudaIpcMemHandle_t mine;
    if (cudaIpcGetMemHandle(&mine, local) != cudaSuccess) {
      cudaGetLastError();
      err = "cudaIpcGetMemHandle failed";
      return -1;
    }
    std::vector<cudaIpcMemHandle_t> all(world);
    if (allgather_host(&mine, all.data(), sizeof(mine), err)) return -1;
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
  void unshare_buffer(void** peers) override {
    for (int r = 0; r < world; ++r)
      if (r != rank && peers[r]) cudaIpcCloseMemHandle(peers[r]);
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

}  // namespace sfl
