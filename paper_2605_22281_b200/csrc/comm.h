// Collectives used by the sharded sketched flexible Golub-Kahan step.
//
// Three implementations of one interface (IpcComm, below, is the third):
//   * NcclComm   — one process per GPU, NCCL over NVLink/NVSwitch.  libnccl is
//                  dlopen'ed on first use (the already-loaded libnccl.so.2, e.g.
//                  PyTorch's, else the system one), so single-GPU use needs no NCCL.
//   * LocalComm  — R ranks inside one process (one host thread per rank), all on
//                  one device: the in-process stand-in used to test the sharded
//                  CUDA path on a single GPU.  Each collective is a host
//                  rendezvous: every rank records an event on its stream, the last
//                  arriving rank makes a comm stream wait for all of them, reduces in
//                  fixed rank order with one kernel, and every rank's stream waits on
//                  the completion event.  No kernel ever waits on another rank.
//   * IpcComm    — one process per rank on one node, host rendezvous in POSIX shared memory and
//                  CUDA-IPC peer memory for the data: the cross-process peer-memory path
//                  without NCCL (NCCL refuses two ranks on one device), used to run the sharded
//                  path and its fused peer-memory collectives across real processes on one GPU.
// All collectives are on fp64 device buffers and are deterministic (fixed
// reduction order; identical bits on every rank).
#pragma once

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace sfl {

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() {}
  // in-place sum / max over ranks of buf[0..count)
  virtual int allreduce(double* buf, size_t count, bool is_max, cudaStream_t s, std::string& err) = 0;
  // recv[r*count .. (r+1)*count) = send of rank r
  virtual int allgather(const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) = 0;
  // recv = sum over ranks of send[rank*count .. (rank+1)*count)
  virtual int reduce_scatter(const double* send, double* recv, size_t count, cudaStream_t s, std::string& err) = 0;
  // blocking host allgather of `bytes` per rank (setup only)
  virtual int allgather_host(const void* send, void* recv, size_t bytes, std::string& err) = 0;
  // Stream-ordered barrier: work issued on s after it starts only when every rank's work issued
  // before its barrier call -- including stores into peer memory -- is complete.
  virtual int barrier(cudaStream_t s, std::string& err) = 0;
  // Peer pointers of a buffer every rank allocated (same role, cudaMalloc base): peers[r] is rank
  // r's buffer addressable from this device (in-process: the raw pointers; NCCL: CUDA IPC).
  virtual int share_buffer(void* local, void** peers, std::string& err) = 0;
  virtual void unshare_buffer(void** peers) { (void)peers; }
  // Host rendezvous around the release of shared buffers (process transports that map peer
  // memory; a no-op where the ranks share an address space or NCCL orders the teardown).
  virtual void release_fence() {}
};

// ---------------------------------------------------------------- NCCL (dlopen)
int nccl_get_unique_id(uint8_t id[128], std::string& err);
Comm* nccl_comm_create(const uint8_t id[128], int rank, int world, int device, std::string& err);

// One-rank self-test of the NCCL transport (every Comm entry, then the same calls captured into a
// CUDA graph and replayed).  0 ok; -2 NCCL unavailable; -3 capture / replay failed; -1 otherwise.
int nccl_selftest(int device, std::string& err);

// ---------------------------------------------------------------- processes + CUDA IPC
// World processes of one node: host rendezvous in the POSIX shared-memory segment `shm_name`
// (created by whichever rank comes first, unlinked once every rank mapped it), data through
// CUDA-IPC peer memory.  Collective over the ranks.
Comm* ipc_comm_create(const char* shm_name, int rank, int world, int device, std::string& err);

// ---------------------------------------------------------------- in-process group
struct LocalGroup;  // shared by the R handles of one group
LocalGroup* local_group_create(int world, int device, std::string& err);
void local_group_release(LocalGroup* g);  // reference counted
Comm* local_comm_create(LocalGroup* g, int rank);

}  // namespace sfl
