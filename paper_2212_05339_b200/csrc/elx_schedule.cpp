// Host-native layout packer and rCache schedule compiler.
//
// elx_layout_pack  : the packing contract of offplan.pack_chunks
//                    (chunking.py:102-138): in-order, first-fit into the open
//                    chunk, close-and-open when the next parameter does not
//                    fit, offsets contiguous from 0, no straddling.
// elx_schedule     : the walk of offplan.simulate (rcache_sim.py:87-199)
//                    compiled into an event program (gathers with their
//                    block/victim and earliest prefetch position, reduces at
//                    reduce_after), plus the SimReport unit counters.
//
// Both run once per plan on the host; the runtime replays the events.
#include <algorithm>
#include <limits>
#include <vector>

#include "elx_internal.h"

extern "C" int elx_layout_pack(const int64_t* numel, int32_t n, int64_t chunk_length,
                               int32_t* chunk_of, int64_t* offset, int32_t* n_chunks) {
  elx::clear_error();
  if (chunk_length < 1) return elx::fail(ELX_ERR_VALIDATION, "chunk_length must be >= 1");
  if (n < 0) return elx::fail(ELX_ERR_VALIDATION, "parameter count must be >= 0");
  if (n > 0 && (!numel || !chunk_of || !offset))
    return elx::fail(ELX_ERR_VALIDATION, "null output or input array");
  if (!n_chunks) return elx::fail(ELX_ERR_VALIDATION, "null n_chunks");
  // Feasibility is checked for the whole sequence before any placement, so a
  // failing call leaves the outputs untouched (chunking.py:104-111).
  for (int32_t i = 0; i < n; ++i) {
    if (numel[i] < 1)
      return elx::fail(ELX_ERR_VALIDATION, "parameter #%d: numel must be >= 1", i);
    if (numel[i] > chunk_length)
      return elx::fail(ELX_ERR_CHUNK_TOO_SMALL,
                       "chunk_length %lld cannot hold parameter #%d with numel %lld",
                       (long long)chunk_length, i, (long long)numel[i]);
  }
  int32_t cur = 0;      // id of the open chunk
  int64_t fill = 0;     // elements already placed in it
  bool open = false;
  for (int32_t i = 0; i < n; ++i) {
    if (open && fill + numel[i] > chunk_length) {  // does not fit: close, open next
      ++cur;
      fill = 0;
    }
    open = true;
    chunk_of[i] = cur;
    offset[i] = fill;
    fill += numel[i];
  }
  *n_chunks = open ? cur + 1 : 0;
  return ELX_OK;
}

namespace {

struct Walk {
  int32_t n_fwd = 0;
  std::vector<std::vector<int32_t>> nodes;  // walk position -> sorted unique chunk ids
};

}  // namespace

extern "C" int elx_schedule(int32_t n_nodes, const int32_t* node_ptr, const int32_t* node_chunks,
                            int32_t n_chunks, int32_t n_block, const uint8_t* cpu_home,
                            elx_event* events, int64_t events_cap, int64_t* n_events,
                            elx_sim_counters* counters) {
  elx::clear_error();
  if (n_block < 1) return elx::fail(ELX_ERR_VALIDATION, "n_block must be >= 1");
  if (n_nodes < 0 || n_chunks < 0) return elx::fail(ELX_ERR_VALIDATION, "negative sizes");
  if (!node_ptr || !n_events || !counters) return elx::fail(ELX_ERR_VALIDATION, "null argument");
  if (n_chunks > 0 && !cpu_home) return elx::fail(ELX_ERR_VALIDATION, "null cpu_home");

  Walk w;
  w.n_fwd = n_nodes;
  w.nodes.resize(2 * (size_t)n_nodes);
  size_t working = 0;
  std::vector<char> appears(n_chunks, 0);
  for (int32_t i = 0; i < n_nodes; ++i) {
    if (node_ptr[i + 1] < node_ptr[i]) return elx::fail(ELX_ERR_VALIDATION, "node_ptr not monotone");
    std::vector<int32_t> ids(node_chunks + node_ptr[i], node_chunks + node_ptr[i + 1]);
    for (int32_t c : ids)
      if (c < 0 || c >= n_chunks)
        return elx::fail(ELX_ERR_VALIDATION, "node %d references chunk id %d outside [0, %d)", i, c,
                         n_chunks);
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    for (int32_t c : ids) appears[c] = 1;
    working = std::max(working, ids.size());
    w.nodes[i] = ids;
    w.nodes[2 * (size_t)n_nodes - 1 - i] = ids;  // backward = reversed forward
  }
  if ((size_t)n_block < working)
    return elx::fail(ELX_ERR_INFEASIBLE_CACHE,
                     "n_block=%d is below the working set of %zu chunks required by a single "
                     "coarse node",
                     n_block, working);

  const int32_t W = 2 * n_nodes;
  // reduce position (backward index) = last backward position touching c.
  std::vector<int32_t> reduce_at(n_chunks, -1);
  for (int32_t b = 0; b < n_nodes; ++b)
    for (int32_t c : w.nodes[n_nodes + b]) reduce_at[c] = b;

  // Occurrence lists for farthest-next-use.
  std::vector<std::vector<int32_t>> occ(n_chunks);
  for (int32_t p = 0; p < W; ++p)
    for (int32_t c : w.nodes[p]) occ[c].push_back(p);
  std::vector<size_t> occ_head(n_chunks, 0);
  const int64_t kNever = std::numeric_limits<int64_t>::max();
  auto next_use = [&](int32_t c) -> int64_t {
    return occ_head[c] < occ[c].size() ? (int64_t)occ[c][occ_head[c]] : kNever;
  };

  std::vector<int32_t> block_of(n_chunks, -1);
  std::vector<char> pinned(n_chunks, 0), pinned_at_prev_start(n_chunks, 0), gathered(n_chunks, 0);
  std::vector<char> in_needed(n_chunks, 0), in_prev_needed(n_chunks, 0);
  std::vector<int32_t> free_blocks;
  for (int32_t b = n_block - 1; b >= 0; --b) free_blocks.push_back(b);  // pop_back -> lowest id
  std::vector<int32_t> resident;  // unordered set of resident chunk ids
  std::vector<int32_t> prev_needed;

  elx_sim_counters cnt{};
  cnt.working_set = (int64_t)working;
  int64_t ne = 0;
  auto emit = [&](const elx_event& e) -> bool {
    if (events && ne < events_cap) events[ne] = e;
    ++ne;
    return true;
  };

  // Prefetch horizon: a gather may be issued as soon as (a) its block's
  // previous owner (the victim) was used for the last time before the
  // eviction — after its release if it was pinned, since a release happens
  // at a needed position — and (b) the chunk itself was last evicted.
  std::vector<int32_t> last_needed(n_chunks, -1), last_evicted(n_chunks, -1);
  std::vector<char> pinned_at_start(n_chunks, 0);
  for (int32_t p = 0; p < W; ++p) {
    const bool backward = p >= n_nodes;
    const int32_t bpos = p - n_nodes;
    const auto& needed = w.nodes[p];
    pinned_at_start = pinned;  // state before this position's pin update
    for (int32_t c : needed) {
      in_needed[c] = 1;
      ++occ_head[c];  // consume this occurrence (rcache_sim.py:134-135)
    }
    for (int32_t c : needed) {  // sorted ascending (rcache_sim.py:137)
      if (block_of[c] >= 0) continue;
      int32_t victim = -1, blk;
      if ((int32_t)resident.size() >= n_block) {
        int64_t best_nu = -1;
        for (int32_t r : resident) {
          if (in_needed[r] || pinned[r]) continue;
          const int64_t nu = next_use(r);
          if (victim < 0 || nu > best_nu || (nu == best_nu && r < victim)) {
            victim = r;
            best_nu = nu;
          }
        }
        if (victim < 0)
          return elx::fail(ELX_ERR_INFEASIBLE_CACHE,
                           "pinned chunks fill all %d blocks at backward position %d; the trace "
                           "cannot execute with this n_block",
                           n_block, bpos);
        blk = block_of[victim];
        block_of[victim] = -1;
        last_evicted[victim] = p;
        resident.erase(std::find(resident.begin(), resident.end(), victim));
      } else {
        blk = free_blocks.back();
        free_blocks.pop_back();
      }
      block_of[c] = blk;
      resident.push_back(c);
      ++cnt.gather_ops;
      if (gathered[c]) ++cnt.replaced_ops;
      gathered[c] = 1;
      if (cpu_home[c]) ++cnt.c2g_units;
      int32_t issue = 0;
      if (victim >= 0) issue = std::max(issue, last_needed[victim] + 1);
      if (last_evicted[c] >= 0) issue = std::max(issue, last_evicted[c]);
      issue = std::min(issue, p);
      emit(elx_event{ELX_EV_GATHER, p, c, blk, victim, issue});
    }
    cnt.peak_rcache_blocks = std::max<int64_t>(cnt.peak_rcache_blocks, (int64_t)resident.size());
    if (backward) {
      for (int32_t c : needed) pinned[c] = 1;
      for (int32_t c : needed) {
        if (reduce_at[c] == bpos) {
          ++cnt.reduce_ops;
          if (cpu_home[c]) ++cnt.g2c_units;
          pinned[c] = 0;
          emit(elx_event{ELX_EV_REDUCE, p, c, block_of[c], -1, p});
        }
      }
    }
    for (int32_t c : prev_needed) in_prev_needed[c] = 0;
    for (int32_t c : needed) {
      in_needed[c] = 0;
      in_prev_needed[c] = 1;
      last_needed[c] = p;
    }
    prev_needed = needed;
    pinned_at_prev_start = pinned_at_start;
  }
  *n_events = ne;
  *counters = cnt;
  if (events && ne > events_cap)
    return elx::fail(ELX_ERR_VALIDATION, "event capacity %lld below required %lld",
                     (long long)events_cap, (long long)ne);
  (void)appears;
  return ELX_OK;
}
