// augment.hpp — host online augmentation (Alg. 2; pseudo shuffle
// P:198-199). Multi-threaded C++17; independent of oracle/.
#pragma once
#include <cstdint>
#include <vector>

#include "host_graph.hpp"

namespace gv {

struct WalkTables {
  const HostGraph* g = nullptr;
  Arr<ProbAlias> departure;  // over nodes, weight = degree
  Arr<ProbAlias> edge;       // per CSR entry: the row's neighbour table (local slots)
};

int build_walk_tables(const HostGraph& g, int threads, WalkTables* t);

// Fills out[2*count] with `threads` pseudo-shuffled walk segments (R-AUG).
// Thread t owns [count*t/threads, count*(t+1)/threads). relabel (nullable):
// ids are emitted as relabel[id] (the relabelled pool id space).
void augment(const WalkTables& t, uint32_t walk_len, uint32_t s, uint32_t threads,
             uint64_t count, uint64_t seed, uint32_t* out, const uint32_t* relabel = nullptr);

}  // namespace gv
