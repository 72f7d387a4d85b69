// ipc.cpp — shared-memory handshake segment of the CUDA-IPC transport.
#include "ipc.hpp"

#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>

namespace gv {

IpcShm* ipc_open(const uint8_t id[128], std::string* name, std::string* err) {
  // FNV-1a of the id names the segment (all ranks share the id)
  uint64_t h = 1469598103934665603ull;
  for (int k = 0; k < 128; ++k) h = (h ^ id[k]) * 1099511628211ull;
  char buf[64];
  std::snprintf(buf, sizeof(buf), "/gv_ipc_%016llx", static_cast<unsigned long long>(h));
  *name = buf;
  const int fd = shm_open(buf, O_CREAT | O_RDWR, 0600);
  if (fd < 0) {
    *err = std::string("shm_open failed for ") + buf;
    return nullptr;
  }
  if (ftruncate(fd, sizeof(IpcShm)) != 0) {
    close(fd);
    *err = "ftruncate of the IPC segment failed";
    return nullptr;
  }
  void* p = mmap(nullptr, sizeof(IpcShm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    *err = "mmap of the IPC segment failed";
    return nullptr;
  }
  return static_cast<IpcShm*>(p);  // a fresh segment is zero-filled
}

void ipc_close(IpcShm* shm, const std::string& name, bool unlink) {
  if (shm) munmap(shm, sizeof(IpcShm));
  if (unlink && !name.empty()) shm_unlink(name.c_str());
}

bool ipc_wait(const std::atomic<uint64_t>& v, uint64_t target, double timeout_s) {
  if (v.load(std::memory_order_acquire) >= target) return true;
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t spin = 0;; ++spin) {
    if (v.load(std::memory_order_acquire) >= target) return true;
    if ((spin & 1023) == 1023) {
      const double dt =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (dt > timeout_s) return false;
      // short waits spin (step handshakes are microseconds apart); long ones
      // (a peer preparing the graph) sleep instead of burning a core
      if (dt > 0.01) usleep(100);
      else sched_yield();
    }
  }
}

}  // namespace gv
