// graph_share.hpp — the node-shared host graph of multi-process runs.
//
// Every rank of Alg. 3 needs the same host-side preparation of
// the graph: the CSR and degrees (augmentation), the zig-zag
// partition, the partitions' negative alias tables and the
// walk tables. On the Friendster-shaped graph that is ~46 GB and
// ~40 s of 16 host threads — per rank if each process prepared it. Instead
// rank 0 prepares it once and copies it into ONE POSIX shared-memory segment;
// every rank of the node (rank 0 included) then views its arrays there,
// read-only, and uploads its device tables from the shared copy
// (DESIGN.md §7).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>

#include "augment.hpp"
#include "host_graph.hpp"

namespace gv {

struct GraphParts {
  HostGraph* graph;
  Partitioning* part;
  Arr<ProbAlias>* nalias;  // negative tables, relabelled order
  WalkTables* walks;
};

struct SharedMapping {
  void* base = nullptr;
  size_t bytes = 0;
};

// Rank 0: copies the prepared parts into segment `name` (created), then
// re-points every Arr of `p` at the segment (its own storage is freed).
int graph_share_publish(const std::string& name, GraphParts p, SharedMapping* map,
                        std::string* err);
// Other ranks: maps segment `name` read-only and points the Arrs of `p` at it.
int graph_share_attach(const std::string& name, GraphParts p, SharedMapping* map,
                       std::string* err);
void graph_share_unmap(SharedMapping* map);
void graph_share_unlink(const std::string& name);

}  // namespace gv
