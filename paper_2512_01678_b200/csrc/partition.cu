// Alg. 4 partitioners, host C++: Phase II component
// bin packing, Phase III load-aware greedy, the relabelling that makes each rank's nodes a
// contiguous id range (so D1-D4 and the NCCL halo path apply unchanged), and the partition
// statistics the cost model of P:545-569 is written in (Σ d̃ per rank = SpMM work, distinct
// ghosts = halo rows, cut entries).  Phase I (METIS) is out of scope.  Reading R9: every sort
// and argmin breaks ties towards the smaller node id / lower rank, so results are bit-exact
// with the oracle.
#include <algorithm>
#include <functional>
#include <queue>
#include <utility>
#include <vector>

#include "internal.cuh"

namespace {

using Load = std::pair<int64_t, int32_t>;  // (weight, rank): the min-heap pops the lighter, then lower rank
using MinHeap = std::priority_queue<Load, std::vector<Load>, std::greater<Load>>;

MinHeap empty_bins(int32_t world) {
  MinHeap h;
  for (int32_t r = 0; r < world; ++r) h.push({0, r});
  return h;
}

}  // namespace

using namespace mph;

extern "C" int mph_partition_greedy(const int64_t* row_ptr_h, int32_t N, int32_t world, int32_t* part_h,
                                    int64_t* load_h) {
  if (!row_ptr_h || !part_h || world < 1 || N < 0) return fail(MPH_EINVAL, "partition_greedy arguments");
  // Ã's row length is d̃ = deg(v) + 1: sort by deg descending, ties by id (stable sort)
  std::vector<int32_t> order((size_t)N);
  for (int32_t v = 0; v < N; ++v) order[v] = v;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return row_ptr_h[a + 1] - row_ptr_h[a] > row_ptr_h[b + 1] - row_ptr_h[b];
  });
  MinHeap bins = empty_bins(world);
  for (int32_t v : order) {
    Load b = bins.top();
    bins.pop();
    part_h[v] = b.second;
    b.first += row_ptr_h[v + 1] - row_ptr_h[v];  // deg(v) + 1
    bins.push(b);
  }
  if (load_h) {
    while (!bins.empty()) {
      load_h[bins.top().second] = bins.top().first;
      bins.pop();
    }
  }
  return MPH_OK;
}

extern "C" int mph_partition_components(const int64_t* row_ptr_h, const int32_t* col_idx_h, int32_t N, int32_t world,
                                        int32_t* part_h, int32_t* n_comp_h) {
  if (!row_ptr_h || !col_idx_h || !part_h || world < 1 || N < 0) return fail(MPH_EINVAL, "partition_components arguments");
  // BFS; components numbered by their smallest node
  std::vector<int32_t> comp((size_t)N, -1), queue;
  std::vector<int64_t> size;
  queue.reserve(1024);
  for (int32_t s = 0; s < N; ++s) {
    if (comp[s] >= 0) continue;
    const int32_t c = (int32_t)size.size();
    comp[s] = c;
    int64_t cnt = 0;
    queue.assign(1, s);
    while (!queue.empty()) {
      const int32_t u = queue.back();
      queue.pop_back();
      ++cnt;
      for (int64_t e = row_ptr_h[u]; e < row_ptr_h[u + 1]; ++e) {
        const int32_t v = col_idx_h[e];
        if (v < 0 || v >= N) return fail(MPH_EINVAL, "partition_components: column %d out of range", v);
        if (comp[v] < 0) {
          comp[v] = c;
          queue.push_back(v);
        }
      }
    }
    size.push_back(cnt);
  }
  const int32_t nc = (int32_t)size.size();
  if (n_comp_h) *n_comp_h = nc;
  if (nc <= 1) return MPH_OK;  // connected: Alg. 4 falls through to Phase III, part untouched
  std::vector<int32_t> order((size_t)nc);
  for (int32_t c = 0; c < nc; ++c) order[c] = c;
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return size[a] > size[b]; });
  std::vector<int32_t> bin_of((size_t)nc);
  MinHeap bins = empty_bins(world);
  for (int32_t c : order) {  // best fit: the lightest bin
    Load b = bins.top();
    bins.pop();
    bin_of[c] = b.second;
    b.first += size[c];
    bins.push(b);
  }
  for (int32_t v = 0; v < N; ++v) part_h[v] = bin_of[comp[v]];
  return MPH_OK;
}

extern "C" int mph_partition_hierarchical(const int64_t* row_ptr_h, const int32_t* col_idx_h, int32_t N,
                                          int32_t world, int32_t* part_h, int32_t* phase_h) {
  int32_t nc = 0;
  MPH_TRY(mph_partition_components(row_ptr_h, col_idx_h, N, world, part_h, &nc));
  if (nc > 1) {
    // reading R10: keep Phase II only when its bins are balanced (none empty, the largest within
    // 5 % of the mean, in |C| units), else fall through to Phase III (a giant component)
    std::vector<int64_t> load((size_t)world, 0);
    for (int32_t v = 0; v < N; ++v) ++load[part_h[v]];
    const int64_t mx = *std::max_element(load.begin(), load.end());
    const int64_t mn = *std::min_element(load.begin(), load.end());
    if (mn > 0 && 100 * (int64_t)world * mx <= 105 * (int64_t)N) {
      if (phase_h) *phase_h = 2;
      return MPH_OK;
    }
  }
  if (phase_h) *phase_h = 3;
  return mph_partition_greedy(row_ptr_h, N, world, part_h, nullptr);
}

extern "C" int mph_relabel(const int32_t* part_h, int32_t N, int32_t world, int64_t* new_id_h, int64_t* bounds_h) {
  if (!part_h || !new_id_h || !bounds_h || world < 1 || N < 0) return fail(MPH_EINVAL, "relabel arguments");
  std::vector<int64_t> next((size_t)world + 1, 0);
  for (int32_t v = 0; v < N; ++v) {
    if (part_h[v] < 0 || part_h[v] >= world) return fail(MPH_EINVAL, "relabel: part[%d] = %d outside [0, %d)", v,
                                                         part_h[v], world);
    ++next[(size_t)part_h[v] + 1];
  }
  for (int32_t r = 0; r < world; ++r) next[r + 1] += next[r];
  for (int32_t r = 0; r <= world; ++r) bounds_h[r] = next[r];
  for (int32_t v = 0; v < N; ++v) new_id_h[v] = next[part_h[v]]++;  // ascending old id within a rank
  return MPH_OK;
}

extern "C" int mph_partition_stats(const int64_t* row_ptr_h, const int32_t* col_idx_h, int32_t N,
                                   const int32_t* part_h, int32_t world, int64_t* stats_h) {
  if (!row_ptr_h || !col_idx_h || !part_h || !stats_h || world < 1 || N < 0)
    return fail(MPH_EINVAL, "partition_stats arguments");
  std::fill(stats_h, stats_h + 4 * (size_t)world, 0);
  const size_t words = ((size_t)N + 63) / 64;
  std::vector<uint64_t> seen((size_t)world * words, 0);  // ghost bitmap per rank
  for (int32_t v = 0; v < N; ++v) {
    const int32_t r = part_h[v];
    if (r < 0 || r >= world) return fail(MPH_EINVAL, "partition_stats: part[%d] = %d outside [0, %d)", v, r, world);
    stats_h[4 * r + 0] += 1;
    stats_h[4 * r + 1] += row_ptr_h[v + 1] - row_ptr_h[v];
    for (int64_t e = row_ptr_h[v]; e < row_ptr_h[v + 1]; ++e) {
      const int32_t u = col_idx_h[e];
      if (u < 0 || u >= N) return fail(MPH_EINVAL, "partition_stats: column %d out of range", u);
      if (part_h[u] == r) continue;
      stats_h[4 * r + 3] += 1;
      uint64_t& w = seen[(size_t)r * words + (size_t)u / 64];
      const uint64_t bit = 1ull << (u % 64);
      if (!(w & bit)) {
        w |= bit;
        stats_h[4 * r + 2] += 1;
      }
    }
  }
  return MPH_OK;
}
