// graph_share.cpp — the node-shared host graph segment (graph_share.hpp).
#include "graph_share.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/gv.h"

namespace gv {

namespace {

constexpr uint64_t kMagic = 0x47565348524431ull;  // "GVSHRD1"
constexpr int kArrays = 10;

struct Header {
  uint64_t magic;
  uint64_t nv, n, pbits, entries;
  uint64_t off[kArrays];    // byte offset of each array in the segment
  uint64_t count[kArrays];  // elements of each array
};

// fallback location of segment `name` (a POSIX shm name starts with '/')
std::string share_file(const std::string& name) {
  const char* dir = getenv("GV_SHARE_DIR");
  std::string d = dir && *dir ? dir : "/tmp";
  return d + "/gv_share" + (name.empty() || name[0] != '/' ? "_" + name : name.substr(1));
}

size_t align64(size_t x) { return (x + 63) & ~size_t(63); }

// The arrays of the segment, in a fixed order: element size and the Arr.
struct Slot {
  size_t elem;
  void (*view)(const GraphParts&, const void*, size_t);
  size_t (*count)(const GraphParts&);
  const void* (*data)(const GraphParts&);
};

#define GV_SLOT(T, expr)                                                                     \
  Slot {                                                                                     \
    sizeof(T), [](const GraphParts& p, const void* d, size_t n) {                            \
      (expr).view(static_cast<const T*>(d), n);                                              \
    },                                                                                       \
        [](const GraphParts& p) -> size_t { return (expr).size(); },                         \
        [](const GraphParts& p) -> const void* { return (expr).data(); }                     \
  }

const Slot kSlots[kArrays] = {
    GV_SLOT(uint64_t, p.graph->off),      GV_SLOT(uint32_t, p.graph->nbr),
    GV_SLOT(double, p.graph->deg),        GV_SLOT(uint32_t, p.part->perm),
    GV_SLOT(uint32_t, p.part->inv_perm),  GV_SLOT(uint64_t, p.part->off),
    GV_SLOT(uint32_t, p.part->packed),    GV_SLOT(ProbAlias, (*p.nalias)),
    GV_SLOT(ProbAlias, p.walks->departure), GV_SLOT(ProbAlias, p.walks->edge),
};
#undef GV_SLOT

void set_views(const GraphParts& p, const Header* h, const char* base) {
  for (int k = 0; k < kArrays; ++k) kSlots[k].view(p, base + h->off[k], h->count[k]);
  p.walks->g = p.graph;
}

}  // namespace

int graph_share_publish(const std::string& name, GraphParts p, SharedMapping* map,
                        std::string* err) {
  Header h{};
  h.magic = kMagic;
  h.nv = p.graph->nv;
  h.n = p.part->n;
  h.pbits = p.part->pbits;
  h.entries = p.graph->nbr.size();
  size_t at = align64(sizeof(Header));
  for (int k = 0; k < kArrays; ++k) {
    h.off[k] = at;
    h.count[k] = kSlots[k].count(p);
    at = align64(at + h.count[k] * kSlots[k].elem);
  }
  // POSIX shared memory (tmpfs) when it has room, else a file under
  // GV_SHARE_DIR (default /tmp): a container's /dev/shm is often 64 MB.
  // posix_fallocate reserves every page up front, so a full tmpfs is an
  // error here instead of a SIGBUS while copying.
  int fd = shm_open(name.c_str(), O_CREAT | O_RDWR | O_TRUNC, 0600);
  if (fd >= 0 && posix_fallocate(fd, 0, static_cast<off_t>(at)) != 0) {
    close(fd);
    shm_unlink(name.c_str());
    fd = -1;
  }
  if (fd < 0) {
    const std::string path = share_file(name);
    fd = open(path.c_str(), O_CREAT | O_RDWR | O_TRUNC, 0600);
    if (fd < 0) {
      *err = "cannot create the shared graph segment (/dev/shm or " + path + ")";
      return GV_ERR_NOMEM;
    }
    if (posix_fallocate(fd, 0, static_cast<off_t>(at)) != 0) {
      close(fd);
      unlink(path.c_str());
      *err = "no room for the shared graph segment (" + std::to_string(at >> 20) +
             " MiB) in /dev/shm or " + path;
      return GV_ERR_NOMEM;
    }
  }
  void* base = mmap(nullptr, at, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (base == MAP_FAILED) {
    graph_share_unlink(name);
    *err = "mmap of the shared graph segment failed";
    return GV_ERR_NOMEM;
  }
  char* b = static_cast<char*>(base);
  for (int k = 0; k < kArrays; ++k) {
    // the large arrays are copied by several threads (tmpfs page faults)
    const char* src = static_cast<const char*>(kSlots[k].data(p));
    const size_t bytes = h.count[k] * kSlots[k].elem;
    parallel_for(bytes, 16, [&](uint64_t s, uint64_t e) { std::memcpy(b + h.off[k] + s, src + s, e - s); });
  }
  std::memcpy(b, &h, sizeof(h));
  mprotect(base, at, PROT_READ);
  set_views(p, &h, b);
  map->base = base;
  map->bytes = at;
  return GV_OK;
}

int graph_share_attach(const std::string& name, GraphParts p, SharedMapping* map,
                       std::string* err) {
  int fd = shm_open(name.c_str(), O_RDONLY, 0600);
  if (fd < 0) fd = open(share_file(name).c_str(), O_RDONLY);
  if (fd < 0) {
    *err = "shm_open failed for the shared graph segment " + name;
    return GV_ERR_COMM;
  }
  struct stat sb;
  if (fstat(fd, &sb) != 0 || static_cast<size_t>(sb.st_size) < sizeof(Header)) {
    close(fd);
    *err = "the shared graph segment is truncated";
    return GV_ERR_COMM;
  }
  void* base = mmap(nullptr, sb.st_size, PROT_READ, MAP_SHARED, fd, 0);
  close(fd);
  if (base == MAP_FAILED) {
    *err = "mmap of the shared graph segment failed";
    return GV_ERR_NOMEM;
  }
  const Header* h = static_cast<const Header*>(base);
  if (h->magic != kMagic || h->nv != p.graph->nv || h->n != p.part->n) {
    munmap(base, sb.st_size);
    *err = "the shared graph segment does not match this context (num_nodes / n_partitions)";
    return GV_ERR_INVALID_ARG;
  }
  p.part->pbits = static_cast<uint32_t>(h->pbits);
  set_views(p, h, static_cast<const char*>(base));
  map->base = base;
  map->bytes = sb.st_size;
  return GV_OK;
}

void graph_share_unmap(SharedMapping* map) {
  if (map->base) munmap(map->base, map->bytes);
  map->base = nullptr;
  map->bytes = 0;
}

void graph_share_unlink(const std::string& name) {
  shm_unlink(name.c_str());
  unlink(share_file(name).c_str());
}

}  // namespace gv
