// ipc.hpp — CUDA-IPC transport between the ranks of one node (world_size > 1).
//
// Each rank is a process driving one GPU (or several processes sharing one
// GPU, as in the single-GPU tests). Device buffers and events are exported
// with cudaIpcGet{Mem,Event}Handle; peers map them and pull data with
// cudaMemcpyAsync (copy engines over NVLink/NVSwitch when the peers are on
// different GPUs). The host-side handshake that makes a cross-process
// cudaStreamWaitEvent safe ("the peer has RECORDED the event for step g")
// goes through a POSIX shared-memory segment of per-rank epoch counters.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

namespace gv {

constexpr int kIpcMaxRanks = 16;
constexpr int kIpcMaxBins = 64 * 64 + 2;
constexpr int kIpcEvRing = 4;    // per-step events are a ring: slot g % 4
constexpr int kIpcSlotRing = 64;
constexpr int kIpcStatRing = 4;  // per-pool statistics: slot e % 4

struct IpcRankShm {
  cudaIpcMemHandle_t ctx_handle;          // context slots buffer
  cudaIpcMemHandle_t blocks_handle;       // receive buffer: my block rows of the pool
  uint64_t blocks_gen;                    // bumped when blocks_handle changes
  cudaIpcEventHandle_t ev_pull[2];        // "placed my samples of pool e" (slot e % 2)
  cudaIpcEventHandle_t ev_first[kIpcEvRing];  // "block 0 of global step g done" (slot g % 4)
  cudaIpcEventHandle_t ev_rot[kIpcEvRing];    // "pulled my rotation of step g" (slot g % 4)
  uint32_t first_slot[kIpcSlotRing];      // context slot of send_part at step g (g % 64)
  uint64_t counts[2][kIpcMaxBins];        // block offsets + error flag of pool e (e % 2)
  double stats[kIpcStatRing][5];          // ms total/bucket/exchange/sgd/rotate of pool e
  std::atomic<uint64_t> counts_epoch;     // e + 1: counts/blocks of pool e published
  std::atomic<uint64_t> pull_epoch;       // e + 1: ev_pull of pool e recorded
  std::atomic<uint64_t> recv_epoch;       // e + 1: receive buffer of pool e ready (handle current)
  std::atomic<uint64_t> first_epoch;      // g + 1: ev_first of step g recorded
  std::atomic<uint64_t> rot_epoch;        // g + 1: ev_rot of step g recorded
  std::atomic<uint64_t> joined;           // init handshake
  std::atomic<uint64_t> stats_epoch;      // e + 1: stats of pool e published
  std::atomic<uint64_t> closed;           // 1: streams drained in gv_destroy (no more pulls)
  char pad[64];
};

struct IpcShm {
  std::atomic<uint64_t> magic;
  std::atomic<uint64_t> arrived;
  std::atomic<uint64_t> graph_state;  // rank 0's shared graph: 0 preparing, 1 ready, 2 + status failed
  IpcRankShm rank[kIpcMaxRanks];
};

// Opens (creating if needed) the segment named after the 128-byte unique id.
IpcShm* ipc_open(const uint8_t id[128], std::string* name, std::string* err);
void ipc_close(IpcShm* shm, const std::string& name, bool unlink);
// Spin until `v` >= target (with sched_yield); false on timeout.
bool ipc_wait(const std::atomic<uint64_t>& v, uint64_t target, double timeout_s);

}  // namespace gv
