// listorder.cuh — bank-group round-robin order of the stored neighbour lists (a permutation only).
//
// The pair kernels gather each list entry's window slot (float4 = 16 B) from shared memory; the 8
// lanes of a quarter-warp read their k-th entries in one access, which is conflict-free only when
// the 8 slots fall in distinct 16-B bank groups (slot mod 8).  In the filter's candidate order the
// groups of different lanes are unrelated, and 55 % of the rates kernels' shared-memory wavefronts
// are bank conflicts (profiles/r1m_ncu_full_bed32M.txt).  This pass re-orders every list so that
// entry k of particle i lies in group (g_i + k) mod 8 for as long as i has entries of that group
// left (exhausted groups are skipped, round by round).  g_i = i's rank in its tile column: the lanes
// of a quarter-warp hold consecutive particles of one tile column, so they start in distinct groups
// and stay apart, and g_i is the same on every slab (slabs split x; the rank depends on the column's
// cells only), which keeps slabs bit-identical to one GPU (measured: i mod 8, not slab-invariant,
// −1.54/−1.44 ms in the rates kernels; the rank inside the cell −1.39/−1.31).  The neighbour SET
// is unchanged; the summation order of the pair loops becomes this fixed permutation of the
// candidate order (reading A34).  Runs after the filter at rebuild steps of Alg. 2.
#pragma once
#include "common.cuh"
#include "tiles.cuh"

namespace crmk {

constexpr int RR_THREADS = 128;

// group of entry e relative to the particle's starting group g (entries are 16 x slot when the
// window is staged; in global mode the plain offset: any permutation is valid there)
__device__ __forceinline__ uint32_t rr_class(uint32_t e, uint32_t g) { return ((e >> 4) - g) & 7u; }

// one thread per list row; per-thread column of cap 16-bit entries in shared memory (buf[pos][tid])
__global__ void __launch_bounds__(RR_THREADS) k_list_rr(int nrows, Grid grid, const uint32_t* __restrict__ cell_of,
                                                        const uint32_t* __restrict__ cell_start,
                                                        uint16_t* __restrict__ list,
                                                        const uint32_t* __restrict__ nlist, ListShape ls) {
  extern __shared__ uint16_t rr_buf[];
  const int i = blockIdx.x * RR_THREADS + threadIdx.x;
  // rows with lists: the particles sorted into cells at this rebuild (slabs: ghosts of the previous
  // step and emigrants sit behind them with stale rows; Alg. 3: the frozen inactive tail)
  if (i >= nrows || (uint32_t)i >= cell_start[grid.M]) return;
  const uint32_t cell = cell_of[i];
  if (cell >= grid.M) return;
  const uint32_t n = min(nlist[i], (uint32_t)ls.cap);
  if (n < 2) return;
  // i's rank in its tile column (the cells of its (x, y) column from z = TZ * floor(cz / TZ) up):
  // the rates kernels give consecutive particles of a tile column to consecutive lanes
  const uint32_t cz = cell % (uint32_t)grid.dims[2];
  const uint32_t g = ((uint32_t)i - cell_start[cell - cz % (uint32_t)TZ]) & 7u;
  const uint32_t nch = (n + 7) >> 3;
  const uint4* L = reinterpret_cast<const uint4*>(list);
  // pass 1: entries per group (8 byte counters; n <= cap <= 255, checked on the host)
  unsigned long long cnt = 0;
  for (uint32_t c = 0; c < nch; ++c) {
    const uint4 v = L[(size_t)c * ls.stride + i];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (c * 8 + e < n) cnt += 1ull << (8 * rr_class(list_entry(v, e), g));
  }
  const unsigned long long start = cnt * 0x0101010101010100ull;   // exclusive prefix per byte
  // pass 2: counting sort by group into the thread's shared-memory column (order kept inside a group)
  unsigned long long pos = start;
  uint32_t fill = 0;
  for (uint32_t c = 0; c < nch; ++c) {
    const uint4 v = L[(size_t)c * ls.stride + i];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t k = c * 8 + e, x = list_entry(v, e);
      if (k < n) {
        const uint32_t sh = 8 * rr_class(x, g);
        rr_buf[(size_t)((pos >> sh) & 0xffu) * RR_THREADS + threadIdx.x] = (uint16_t)x;
        pos += 1ull << sh;
      } else if (k == n) {
        fill = x;   // the padding entry (zero weight) of the last chunk
      }
    }
  }
  // emission, round by round over the groups g, g+1, ... (same thread: every read precedes the writes)
  // (measured: placing each entry directly at its round-robin position, computed with byte-SIMD
  //  min/compare/dot products, 9.4 ms against 8.8)
  uint32_t cj[8], sj[8], mx = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    cj[j] = (uint32_t)(cnt >> (8 * j)) & 0xffu;
    sj[j] = (uint32_t)(start >> (8 * j)) & 0xffu;
    mx = max(mx, cj[j]);
  }
  ListWriter w;
  w.init(list, (size_t)i, ls);
  for (uint32_t r = 0; r < mx; ++r) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (r < cj[j]) w.push(rr_buf[(size_t)(sj[j] + r) * RR_THREADS + threadIdx.x]);
  }
  w.flush(fill);
}

}  // namespace crmk
