// tiles.cuh — shared-memory-staged cell tiles for the fused neighbour filter and pair loops.
//
// A tile is TX x TY cell columns x TZ cells along z.  With the B3 cell order (z fastest) the
// particles of one column segment are one contiguous index range, so a tile's "window" — every
// particle of the 27-cell neighbourhoods of the tile's particles — is WR = (TX+2)(TY+2)
// contiguous runs.  One CTA per tile stages the window's 56-B states into shared memory once,
// filters candidates there (Alg. 1) and runs the pair loops from shared memory.
// Neighbour lists store 16-bit window BYTE offsets (list entry = 16 x position in the tile window,
// so a pair loop addresses the staged float4 arrays with no index arithmetic; global mode stores the
// plain position, windows up to 65535 particles), per particle
// contiguous (cap entries, 16-B aligned chunks of 8), read and written with 16-B vector accesses.  Windows larger than WMAX are read from global memory instead
// (same list format, slower; "global mode").
#pragma once
#include <cuda_pipeline.h>

#include "common.cuh"

namespace crmk {

constexpr int TX = 2, TY = 2, TZ = 4;
constexpr int WRX = TX + 2, WRY = TY + 2, WR = WRX * WRY;   // 16 window runs
constexpr int NCOL = TX * TY;                               // i columns per tile
#ifndef CRM_TILE_THREADS
#define CRM_TILE_THREADS 384
#endif
constexpr int TILE_THREADS = CRM_TILE_THREADS;
// 2 CTAs of 384 threads per SM (80 registers; the pair loops do not spill).  A tile holds 250-330
// particles on the C5 lattice (2h = 2.6 d0 cells alias the lattice: up to 396 with walls): with
// 288 threads a quarter of the tiles ran a second round for a few particles and took twice as long
// (measured: 288 -> 384 threads, rates kernels -14 %; 448 threads spill and are slower)
#define TILE_BOUNDS __launch_bounds__(TILE_THREADS, 2)
#ifndef CRM_BCE_THREADS
#define CRM_BCE_THREADS 320
#endif
// the BCE kernels' CTAs (2 per SM: the same window); 320 threads leave 96 registers and no spills
// (measured: k_bce_A/B 0.75 -> 0.70 ms against 384; 256: 0.73, 192: 0.90)
constexpr int BCE_THREADS = CRM_BCE_THREADS;
#define BCE_BOUNDS __launch_bounds__(BCE_THREADS, 2)
#ifndef CRM_WMAX
#define CRM_WMAX 1968
#endif
constexpr int WMAX = CRM_WMAX;   // staged window capacity (particles): 1920 sent 6 % of the C5 tiles to global mode

// tile geometry shared by every tile kernel (the window arrays follow in the derived structs)
struct TileHead {
  uint32_t run_start[WR];       // first global index of each window run
  uint32_t run_base[WR + 1];    // window offset of each run (prefix of lengths)
  uint32_t wcs[WR][TZ + 3];     // cellStart of the run's cells zlo..zhi, plus the end
  uint32_t col_start[NCOL];     // first i of each tile column
  uint32_t col_pref[NCOL + 1];  // prefix of i counts
  int zlo, zhi, staged;
  int X0, Y0;
  float ox, oy, oz;             // tile origin: pair loops use positions relative to it
};

// the rates / BCE kernels stage the whole 56-B state of the window
struct TileSmem : TileHead {
  float4 P[WMAX];
  float4 U[WMAX];
  float4 S1[WMAX];
  float2 S2[WMAX];
};

struct TileGeom {
  int X0, Y0, z0, z1, zlo, zhi;
};

__host__ __device__ inline int tiles_x(const Grid& g) { return (g.dims[0] + TX - 1) / TX; }
__host__ __device__ inline int tiles_y(const Grid& g) { return (g.dims[1] + TY - 1) / TY; }
__host__ __device__ inline int tiles_z(const Grid& g) { return (g.dims[2] + TZ - 1) / TZ; }
__host__ inline long long num_tiles(const Grid& g) { return (long long)tiles_x(g) * tiles_y(g) * tiles_z(g); }

__device__ __forceinline__ uint32_t cell_id(const Grid& g, int cx, int cy, int cz) {
  return (uint32_t)cx * (uint32_t)(g.dims[1] * g.dims[2]) + (uint32_t)cy * (uint32_t)g.dims[2] + (uint32_t)cz;
}

__device__ __forceinline__ TileGeom tile_geom(const Grid& g, long long t) {
  const int ntz = tiles_z(g), nty = tiles_y(g);
  TileGeom G;
  const uint32_t t32 = (uint32_t)t, tq = t32 / (uint32_t)ntz;   // tile indices < 2^32
  const int tz = (int)(t32 - tq * (uint32_t)ntz);
  const int tx = (int)(tq / (uint32_t)nty);
  const int ty = (int)(tq - (uint32_t)tx * (uint32_t)nty);
  G.X0 = tx * TX;
  G.Y0 = ty * TY;
  G.z0 = tz * TZ;
  G.z1 = min(G.z0 + TZ, g.dims[2]);
  G.zlo = max(G.z0 - 1, 0);
  G.zhi = min(G.z1, g.dims[2] - 1);
  return G;
}

// Active domains (Alg. 3): the tiles holding at least one (non-Inactive) particle, appended to
// `list` (absolute tile indices, any order: tiles are independent) with warp-aggregated atomics.
__global__ void k_tile_list(long long ntiles, long long tile_base, Grid g, const uint32_t* __restrict__ cell_start,
                            uint32_t* __restrict__ list, uint32_t* __restrict__ count) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool keep = false;
  if (t < ntiles) {
    const TileGeom G = tile_geom(g, tile_base + t);
    uint32_t n = 0;
    for (int q = 0; q < NCOL; ++q) {
      const int cx = G.X0 + q / TY, cy = G.Y0 + q % TY;
      if (cx < g.dims[0] && cy < g.dims[1]) {
        const uint32_t c0 = cell_id(g, cx, cy, G.z0);
        n += cell_start[c0 + (G.z1 - G.z0)] - cell_start[c0];
      }
    }
    keep = n > 0;
  }
  const unsigned m = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == 0 && m) base = atomicAdd(count, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) list[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)(tile_base + t);
}

// Fill the tile geometry in shared memory (all threads call; contains __syncthreads).
__device__ __forceinline__ void tile_setup(const Grid& g, const TileGeom& G, const uint32_t* __restrict__ cell_start,
                                          TileHead& sm) {
  // warp 0 alone: lane r < 16 reads its run's cell starts; run bases and the tile columns' prefix
  // by shuffle scans (one barrier; measured: a serial thread-0 pass cost ~3 % of a rates kernel)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int nzw = G.zhi - G.zlo + 1;
    uint32_t len = 0, cb = 0, cn = 0;
    if (lane < WR) {
      const int r = lane;
      const int cx = G.X0 - 1 + r / WRY, cy = G.Y0 - 1 + r % WRY;
      const bool valid = cx >= 0 && cx < g.dims[0] && cy >= 0 && cy < g.dims[1];
      const uint32_t c0 = valid ? cell_id(g, cx, cy, G.zlo) : 0u;
      uint32_t first = 0, last = 0;
      // all (at most TZ + 3) cell starts requested at once: one memory round trip instead of a
      // dependent chain (the setup is on every tile kernel's critical path)
      uint32_t v[TZ + 3];
#pragma unroll
      for (int k = 0; k < TZ + 3; ++k) v[k] = (valid && k <= nzw) ? cell_start[c0 + k] : 0u;
#pragma unroll
      for (int k = 0; k < TZ + 3; ++k) {
        if (k <= nzw) sm.wcs[r][k] = v[k];
        if (k == 0) first = v[k];
        if (k == nzw) last = v[k];
        if (k == G.z0 - G.zlo) cb = v[k];
        if (k == G.z1 - G.zlo) cn = v[k];
      }
      sm.run_start[r] = first;
      len = last - first;
      cn -= cb;   // particles of the run's column inside the tile (used for the tile's own columns)
    }
    uint32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane < WR) sm.run_base[lane] = incl - len;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, WR - 1);
    // tile column q = run (1 + q / TY) * WRY + (1 + q % TY)
    const int rq = (1 + (lane & (NCOL - 1)) / TY) * WRY + (1 + (lane & (NCOL - 1)) % TY);
    const uint32_t qb = __shfl_sync(0xffffffffu, cb, rq), qn = __shfl_sync(0xffffffffu, cn, rq);
    uint32_t qincl = lane < NCOL ? qn : 0u;
#pragma unroll
    for (int o = 1; o < NCOL; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, qincl, o);
      if (lane >= o) qincl += v;
    }
    if (lane < NCOL) {
      sm.col_start[lane] = qb;
      sm.col_pref[lane] = qincl - qn;
    }
    if (lane == NCOL - 1) sm.col_pref[NCOL] = qincl;
    if (lane == 0) {
      sm.run_base[WR] = total;
      sm.zlo = G.zlo;
      sm.zhi = G.zhi;
      sm.X0 = G.X0;
      sm.Y0 = G.Y0;
      sm.ox = g.lo[0] + (float)G.X0 * g.s;
      sm.oy = g.lo[1] + (float)G.Y0 * g.s;
      sm.oz = g.lo[2] + (float)G.z0 * g.s;
      sm.staged = total <= (uint32_t)WMAX;
    }
  }
  __syncthreads();
}

// Copy the window of (P,U,S1,S2) into shared memory (only when it fits) with asynchronous
// global->shared copies (LDGSTS): every copy of the block is in flight at once; the caller
// waits with tile_stage_wait() + __syncthreads().
__device__ __forceinline__ void tile_stage(const float4* __restrict__ P, const float4* __restrict__ U,
                                           const float4* __restrict__ S1, const float2* __restrict__ S2, TileSmem& sm) {
  if (!sm.staged) return;
  // one warp per window run (no per-element run search: measured 6 % of a rates kernel's issue)
  const uint32_t lane = threadIdx.x & 31u, nw = blockDim.x >> 5;
  for (uint32_t r = threadIdx.x >> 5; r < (uint32_t)WR; r += nw) {
    const uint32_t b = sm.run_base[r], e = sm.run_base[r + 1];
    const int shift = (int)sm.run_start[r] - (int)b;
    for (uint32_t idx = b + lane; idx < e; idx += 32) {
      const uint32_t gidx = (uint32_t)((int)idx + shift);
      __pipeline_memcpy_async(&sm.P[idx], &P[gidx], sizeof(float4));
      __pipeline_memcpy_async(&sm.U[idx], &U[gidx], sizeof(float4));
      __pipeline_memcpy_async(&sm.S1[idx], &S1[gidx], sizeof(float4));
      __pipeline_memcpy_async(&sm.S2[idx], &S2[gidx], sizeof(float2));
    }
  }
  __pipeline_commit();
}

// BCE kernels: only the cells klo..khi-1 (relative to zlo) of every run, at their usual window
// offsets (the markers' list entries lie within one cell of the markers' cells)
__device__ __forceinline__ void tile_stage_cells(const float4* __restrict__ P, const float4* __restrict__ U,
                                                 const float4* __restrict__ S1, const float2* __restrict__ S2,
                                                 TileSmem& sm, int klo, int khi) {
  if (!sm.staged) return;
  const uint32_t lane = threadIdx.x & 31u, nw = blockDim.x >> 5;
  for (uint32_t r = threadIdx.x >> 5; r < (uint32_t)WR; r += nw) {
    const uint32_t rs = sm.run_start[r], rb = sm.run_base[r];
    const uint32_t b = rb + (sm.wcs[r][klo] - rs), e = rb + (sm.wcs[r][khi] - rs);
    const int shift = (int)rs - (int)rb;
    for (uint32_t idx = b + lane; idx < e; idx += 32) {
      const uint32_t gidx = (uint32_t)((int)idx + shift);
      __pipeline_memcpy_async(&sm.P[idx], &P[gidx], sizeof(float4));
      __pipeline_memcpy_async(&sm.U[idx], &U[gidx], sizeof(float4));
      __pipeline_memcpy_async(&sm.S1[idx], &S1[gidx], sizeof(float4));
      __pipeline_memcpy_async(&sm.S2[idx], &S2[gidx], sizeof(float2));
    }
  }
  __pipeline_commit();
}

__device__ __forceinline__ void tile_stage_wait() { __pipeline_wait_prior(0); }

// Positions are stored compensated, x = hi + lo (hi: the fp32 value the structural rules B1/B2
// use; lo: the rounding remainder kept by the integrator).  The pair loops work in coordinates
// relative to the tile origin, (hi - o) + lo, which keeps ~1e-9 m resolution on metre-scale beds.
__device__ __forceinline__ float4 rel_pos(const float4& hi, const float4& lo, const TileHead& sm) {
  return make_float4((hi.x - sm.ox) + lo.x, (hi.y - sm.oy) + lo.y, (hi.z - sm.oz) + lo.z, hi.w);
}
// the same with lo decoded from the quantised copy in the tag word (common.cuh): what the pair and
// BCE kernels use, from the staged window, with no global lo loads
__device__ __forceinline__ float4 rel_pos_q(const float4& hi, uint32_t tag, const TileHead& sm) {
  return make_float4((hi.x - sm.ox) + loq_value(tag, 0, hi.x), (hi.y - sm.oy) + loq_value(tag, 1, hi.y),
                     (hi.z - sm.oz) + loq_value(tag, 2, hi.z), hi.w);
}

// signed neighbour volume carried in the .w slot of a rates window: +m/rho for fluid, -m/rho for
// markers (A7, A8: markers are ordinary neighbours with V = m/rho0; the sign lets the marker-load
// loop keep fluid neighbours only without reading the tag)
__device__ __forceinline__ float signed_volume(float rho, float tagw, float m) {
  const float V = __fdiv_rn(m, rho);
  return tag_is_bce(tag_of(tagw)) ? -V : V;
}

#ifndef CRM_RELK_UNROLL
#define CRM_RELK_UNROLL 1
#endif
// convert the staged window from absolute hi to relative compensated positions (lo from the staged
// tag words: no global loads; measured: the per-slot lo loads of the previous design held every tile's
// prologue ~1.2 ms per step); TO_V: the rates kernels also replace rho_j by the signed volume V_j (one
// division per staged particle instead of one reciprocal per pair)
constexpr int RELK = (WMAX + TILE_THREADS - 1) / TILE_THREADS;   // window slots per thread (blockDim == TILE_THREADS)
template <bool TO_V>
__device__ __forceinline__ void relativize_apply(TileSmem& sm, float m) {
  if (!sm.staged) return;
  const uint32_t W = sm.run_base[WR];
#if CRM_RELK_UNROLL
#pragma unroll
  for (int k = 0; k < RELK; ++k) {
    const uint32_t idx = threadIdx.x + (uint32_t)k * blockDim.x;
    if (idx < W) {
#else
  for (uint32_t idx = threadIdx.x; idx < W; idx += blockDim.x) {
    {
#endif
      const float tw = sm.U[idx].w;
      float4 p = rel_pos_q(sm.P[idx], tag_of(tw), sm);
      if (TO_V) p.w = signed_volume(p.w, tw, m);
      sm.P[idx] = p;
    }
  }
}
// the BCE kernels' variant (densities kept: the Adami stress needs rho_f) over the staged cells
// klo..khi-1 of every run, one warp per run
__device__ __forceinline__ void tile_relativize_cells(TileSmem& sm, int klo, int khi) {
  if (!sm.staged) return;
  const uint32_t lane = threadIdx.x & 31u, nw = blockDim.x >> 5;
  for (uint32_t r = threadIdx.x >> 5; r < (uint32_t)WR; r += nw) {
    const uint32_t rs = sm.run_start[r], rb = sm.run_base[r];
    const uint32_t b = rb + (sm.wcs[r][klo] - rs), e = rb + (sm.wcs[r][khi] - rs);
    for (uint32_t idx = b + lane; idx < e; idx += 32) sm.P[idx] = rel_pos_q(sm.P[idx], tag_of(sm.U[idx].w), sm);
  }
}
// staged window entries by list entry (byte offset of the float4 slot)
__device__ __forceinline__ float4 win_P(const TileSmem& sm, uint32_t e) {
  return *reinterpret_cast<const float4*>(reinterpret_cast<const char*>(sm.P) + e);
}
__device__ __forceinline__ float4 win_U(const TileSmem& sm, uint32_t e) {
  return *reinterpret_cast<const float4*>(reinterpret_cast<const char*>(sm.U) + e);
}
__device__ __forceinline__ float4 win_S1(const TileSmem& sm, uint32_t e) {
  return *reinterpret_cast<const float4*>(reinterpret_cast<const char*>(sm.S1) + e);
}
__device__ __forceinline__ float2 win_S2(const TileSmem& sm, uint32_t e) {
  return *reinterpret_cast<const float2*>(reinterpret_cast<const char*>(sm.S2) + (e >> 1));
}

// compensated update (hi, lo) += d  (Fast2Sum; |hi| >= |lo + d| for any step an SPH particle takes)
__device__ __forceinline__ void comp_add(float& hi, float& lo, float d) {
  const float y = lo + d;
  const float t = hi + y;
  lo = y - (t - hi);
  hi = t;
}

// global index of a window offset (global mode, where list entries are plain offsets)
__device__ __forceinline__ uint32_t window_to_global(const TileHead& sm, uint32_t off) {
  int r = 0;
#pragma unroll
  for (int k = 1; k < WR; ++k) r += (sm.run_base[k] <= off) ? 1 : 0;
  return sm.run_start[r] + (off - sm.run_base[r]);
}

// tile-local slot t -> (global i, column q)
__device__ __forceinline__ uint32_t tile_particle(const TileHead& sm, uint32_t t, int& q) {
  q = 0;
#pragma unroll
  for (int k = 1; k < NCOL; ++k) q += (sm.col_pref[k] <= t) ? 1 : 0;
  return sm.col_start[q] + (t - sm.col_pref[q]);
}

// candidate window-offset range of run (da, db) for a particle of column q at cell z = cz
__device__ __forceinline__ void cand_range(const TileHead& sm, int q, int da, int db, int cz, uint32_t& ob,
                                           uint32_t& oe, int& r) {
  r = (1 + q / TY + da) * WRY + (1 + q % TY + db);
  const int klo = max(cz - 1, sm.zlo) - sm.zlo;
  const int khi = min(cz + 1, sm.zhi) - sm.zlo + 1;
  const uint32_t rs = sm.run_start[r], rb = sm.run_base[r];
  ob = rb + (sm.wcs[r][klo] - rs);
  oe = rb + (sm.wcs[r][khi] - rs);
}

// 16-bit list writer: entries are collected in a 128-bit funnel-shift register buffer and
// written 8 at a time with one 16-B store (chunk-major layout, see ListShape); the last
// chunk is padded with `fill` (the particle's own window offset: a zero-weight entry), so the
// pair loops read whole 16-B chunks and run without per-entry branches.
// list layout: chunk-major ELL of 16-B chunks (8 entries): chunk c of particle (slot) i at uint4
// index c * stride + i, so the 32 lanes of a warp (consecutive slots) read one chunk each with a
// single coalesced 512-B access; cap entries (cap % 8 == 0) per particle, stride = rows allocated
struct ListShape {
  int cap;
  uint32_t stride;
};

struct ListWriter {
  uint2* cur;        // the next 8-B half-chunk to store (chunk-major layout, see ListShape)
  size_t step;       // from half 1 of chunk c to half 0 of chunk c + 1: 2 * stride - 1 halves
  size_t stride;     // uint4 rows per chunk
  uint32_t b0, b1;   // the last 4 entries (16 bits each, oldest in the low half of b0)
  int k;             // entries found (may exceed cap: overflow is reported by the caller)
  int cap;
  bool closed;       // the list was written whole (padded) by its producer; flush does nothing
  __device__ __forceinline__ void init(uint16_t* list, size_t i, ListShape ls) {
    cur = reinterpret_cast<uint2*>(list) + 2 * i;
    step = 2 * (size_t)ls.stride - 1;
    stride = ls.stride;
    b0 = b1 = 0u;
    k = 0;
    cap = ls.cap;
    closed = false;
  }
  // (measured: 4-entry buffer + 8-B stores with the capacity test only at the store beat the
  //  16-B funnel buffer with a per-entry capacity branch, and one 2-B store per entry; the store
  //  address advances incrementally — recomputing it from k cost 13 instructions per store)
  __device__ __forceinline__ void store(int kk) {   // entries kk - 4 .. kk - 1 are in (b0, b1)
    if (kk <= cap) *cur = make_uint2(b0, b1);
    cur += (kk & 4) ? 1 : step;   // kk % 8 == 4: the second half of the chunk is next
  }
  __device__ __forceinline__ void push(uint32_t off) {
    b0 = __funnelshift_r(b0, b1, 16);
    b1 = __funnelshift_r(b1, off, 16);
    ++k;
    if ((k & 3) == 0) store(k);
  }
  // pad the last chunk of 8 with `fill` (a zero-weight entry); k keeps the unpadded count.  An empty
  // list still gets one chunk of padding: the pair kernels prefetch chunk 0 of every list.
  __device__ __forceinline__ void flush(uint32_t fill) {
    if (closed || k >= cap) return;   // cap % 8 == 0: the stored part ends on a chunk boundary
    int kk = k;
    while ((kk & 7) || kk == 0) {
      b0 = __funnelshift_r(b0, b1, 16);
      b1 = __funnelshift_r(b1, fill, 16);
      ++kk;
      if ((kk & 3) == 0) store(kk);
    }
  }
};

__device__ __forceinline__ uint32_t list_entry(const uint4& v, int e) {
  const uint32_t w = (e < 2) ? v.x : (e < 4) ? v.y : (e < 6) ? v.z : v.w;
  return (e & 1) ? (w >> 16) : (w & 0xffffu);
}

}  // namespace crmk
