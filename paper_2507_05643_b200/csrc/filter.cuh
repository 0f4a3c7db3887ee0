// filter.cuh — Alg. 1 neighbour lists in a kernel of their own.
//
//   k_filter_t  one CTA per cell tile; stages only the window's positions (16 B) and a BCE flag
//               (1 B) per particle — a quarter of the rates kernels' 56-B window — so several CTAs
//               share an SM and the branchy, latency-bound candidate sweep runs at high occupancy
//               instead of inside the register- and shared-memory-limited pair kernels.  Every
//               particle of the tile gets its list: fluid particles all neighbours, markers their
//               fluid neighbours (Adami sums run over fluid only), or all with store_all
//               (debug export).  count_all = |P(i)| for the structure checks.  The tiles that hold
//               markers are appended to `mtiles` for the BCE kernels.
// Runs only at rebuild steps of Alg. 2 (t mod ps_freq == 0); the tile kernels read the lists.
// The predicate is rule B2 on the absolute fp32 positions; the candidate order (runs in (da, db)
// order, offsets ascending) fixes the list order and hence the summation order of the pair loops.
#pragma once
#include "common.cuh"
#include "structure.cuh"
#include "tiles.cuh"

namespace crmk {

// The window is staged as three coordinate arrays (structure of arrays), so one 16-byte load gives
// four candidates' x (or y, z) and the B2 predicate of two candidates runs on the packed f32x2
// FP32 instructions of sm_100 (FADD2/FMUL2/FFMA2: per element the same IEEE round-to-nearest
// results as the scalar instructions, half the issue slots; this kernel is issue-bound).
#ifndef CRM_FILTER_THREADS
#define CRM_FILTER_THREADS 128
#define CRM_FILTER_MINB 5
#endif
constexpr int FILTER_THREADS = CRM_FILTER_THREADS;
constexpr int FMW = 24;   // stored 32-candidate hit masks per particle (more: drained early)

struct FilterSmem : TileHead {
  int mzmin, mzmax;                 // cells z of the tile's markers (min, max)
  alignas(16) float X[WMAX + 40];   // absolute positions (a chunk may read up to 39 slots past a segment)
  float Y[WMAX + 40];
  float Z[WMAX + 40];
  alignas(4) uint8_t bce[WMAX + 40];    // 1 = BCE marker
  // each thread's hit masks (word-major: thread t's word w at [w][t], bank = t) and the window
  // offset of each mask's bit 0; drained into the list once the particle's sweep is complete
  uint32_t mw[FMW][FILTER_THREADS];
  uint16_t wb[FMW][FILTER_THREADS];
};

// positions + flags of the window (LDGSTS for the positions)
__device__ __forceinline__ void filter_stage(const float4* __restrict__ P, const float4* __restrict__ U,
                                             FilterSmem& sm) {
  if (!sm.staged) return;
  const uint32_t lane = threadIdx.x & 31u, nw = blockDim.x >> 5;
  for (uint32_t r = threadIdx.x >> 5; r < (uint32_t)WR; r += nw) {   // one warp per window run
    const uint32_t b = sm.run_base[r], e = sm.run_base[r + 1];
    const int shift = (int)sm.run_start[r] - (int)b;
    for (uint32_t idx = b + lane; idx < e; idx += 32) {
      const uint32_t gidx = (uint32_t)((int)idx + shift);
      const float* pg = reinterpret_cast<const float*>(&P[gidx]);
      __pipeline_memcpy_async(&sm.X[idx], pg + 0, sizeof(float));
      __pipeline_memcpy_async(&sm.Y[idx], pg + 1, sizeof(float));
      __pipeline_memcpy_async(&sm.Z[idx], pg + 2, sizeof(float));
      sm.bce[idx] = tag_is_bce(tag_of(U[gidx].w)) ? 1 : 0;
    }
  }
  __pipeline_commit();
}

// rule B2 for the 8 candidates j .. j + 7 (j % 4 == 0): bit e = "neighbour".  Positions come in
// 16-B loads (4 candidates' x per load), r2 - R2 in packed f32x2, and the bits are the sign bits of
// fl(r2 - R2): for r2 < R2 the exact difference is negative and its rounding stays < 0 (no
// underflow: |r2 - R2| >= ulp(R2) >> FLT_MIN), for r2 >= R2 it is >= +0 — so each bit equals
// (r2 < R2) exactly.  The sign bytes are gathered with byte permutes and packed by one multiply.
// (measured: 54 instructions per group against 67 with 8-B loads and FSETP/SEL per candidate;
//  k_filter 14.05 -> 13.98 ms — the sweep is not where the kernel's issue slots go, the appends are)
__device__ __forceinline__ unsigned long long b2_r2m(unsigned long long x, unsigned long long y, unsigned long long z,
                                                     unsigned long long xi2, unsigned long long yi2,
                                                     unsigned long long zi2, unsigned long long R2x2) {
  const unsigned long long dx = f2_sub(x, xi2), dy = f2_sub(y, yi2), dz = f2_sub(z, zi2);   // x_j - x_i
  return f2_sub(f2_fma(dz, dz, f2_fma(dy, dy, f2_mul(dx, dx))), R2x2);
}
__device__ __forceinline__ uint32_t sign_nibble(unsigned long long d0, unsigned long long d1) {
  // bytes (d0.lo.b3, d0.hi.b3, d1.lo.b3, d1.hi.b3); sign bits at 7, 15, 23, 31
  const uint32_t w = __byte_perm(__byte_perm((uint32_t)d0, (uint32_t)(d0 >> 32), 0x0073),
                                 __byte_perm((uint32_t)d1, (uint32_t)(d1 >> 32), 0x0073), 0x5410);
  return (w & 0x80808080u) * 0x00204081u;   // the 4 bits land at 28..31 (nothing below 24)
}
__device__ __forceinline__ uint32_t b2_group8(const FilterSmem& sm, uint32_t j, unsigned long long xi2,
                                              unsigned long long yi2, unsigned long long zi2,
                                              unsigned long long R2x2) {
  const ulonglong2 xa = *reinterpret_cast<const ulonglong2*>(&sm.X[j]);
  const ulonglong2 ya = *reinterpret_cast<const ulonglong2*>(&sm.Y[j]);
  const ulonglong2 za = *reinterpret_cast<const ulonglong2*>(&sm.Z[j]);
  const ulonglong2 xb = *reinterpret_cast<const ulonglong2*>(&sm.X[j + 4]);
  const ulonglong2 yb = *reinterpret_cast<const ulonglong2*>(&sm.Y[j + 4]);
  const ulonglong2 zb = *reinterpret_cast<const ulonglong2*>(&sm.Z[j + 4]);
  const uint32_t a = sign_nibble(b2_r2m(xa.x, ya.x, za.x, xi2, yi2, zi2, R2x2),
                                 b2_r2m(xa.y, ya.y, za.y, xi2, yi2, zi2, R2x2));
  const uint32_t b = sign_nibble(b2_r2m(xb.x, yb.x, zb.x, xi2, yi2, zi2, R2x2),
                                 b2_r2m(xb.y, yb.y, zb.y, xi2, yi2, zi2, R2x2));
  return (a >> 28) | (b >> 24);
}

// drain the stored masks of this thread (words 0 .. nw-1) into the list, in candidate order; all
// threads of a warp run it once, at the end of their sweeps, so they append in lockstep (the
// k % 4 store points of ListWriter coincide)
template <bool STAGED>
__device__ __forceinline__ void drain_masks(const FilterSmem& sm, int nw, uint32_t nent, ListWriter& w) {
  const uint32_t t = threadIdx.x;
  int wi = 0;
  uint32_t M = nw > 0 ? sm.mw[0][t] : 0u, base = nw > 0 ? sm.wb[0][t] : 0u;
  for (uint32_t e = 0; e < nent; ++e) {
    while (M == 0u) {   // (a thread advances every ~4 entries)
      ++wi;
      M = sm.mw[wi][t];
      base = sm.wb[wi][t];
    }
    const uint32_t off = base + (__ffs(M) - 1);
    M &= M - 1;
    w.push(STAGED ? off << 4 : off);   // list entry: byte offset of the staged slot (global mode: the offset)
  }
}

// Alg. 1 over one contiguous candidate range [ob, oe) of window offsets, skipping offset `self`
// (j != i, A18; ~0u for runs without i): chunks of 32 candidates, a branch-free predicate sweep
// builds a bitmask (and, for marker lists, a mask of the fluid candidates); the masks are stored
// (drain_masks appends their set bits later; a thread whose FMW slots are full drains early).
// (measured round 1: masking i's bit beats splitting its run in two ranges; 64-candidate chunks with
//  64-bit masks cost more in 64-bit bit arithmetic than they save)
template <bool STAGED, bool STORE_BCE>
__device__ __forceinline__ void filter_range(float R2, FilterSmem& sm, const float4* __restrict__ P,
                                             const float4* __restrict__ U, uint32_t ob, uint32_t oe, uint32_t self,
                                             uint32_t gshift, const float4& pi, uint32_t& cnt, int& nw,
                                             uint32_t& nent, ListWriter& w) {
  const unsigned long long xi2 = f2_splat(pi.x), yi2 = f2_splat(pi.y), zi2 = f2_splat(pi.z);
  // staged: chunks start on an aligned slot (vector loads); the slots before ob are masked off
  const unsigned long long R2x2 = f2_splat(R2);
  for (uint32_t base = STAGED ? (ob & ~3u) : ob; base < oe; base += 32) {   // staged: 16-B aligned
    const uint32_t nc = min(32u, oe - base);
    uint32_t m = 0, mf = 0;
    if (STAGED) {
      // groups of 8 with compile-time bit positions; the last group may read up to 7 slots past
      // the segment (inside FilterSmem), masked off below
      for (uint32_t k8 = 0; k8 < nc; k8 += 8) {
        uint32_t gm = 0, gf = 0;
        gm = b2_group8(sm, base + k8, xi2, yi2, zi2, R2x2);
        if (!STORE_BCE) {   // the 8 flags (bytes 0/1) in two 4-B loads, packed to bits by multiplies
          const uint32_t f0 = *reinterpret_cast<const uint32_t*>(&sm.bce[base + k8]);
          const uint32_t f1 = *reinterpret_cast<const uint32_t*>(&sm.bce[base + k8 + 4]);
          const uint32_t fb = ((f0 * 0x01020408u) >> 24) | (((f1 * 0x01020408u) >> 20) & 0xf0u);
          gf = gm & ~fb;
        }
        m |= gm << k8;
        mf |= gf << k8;
      }
    } else {
#pragma unroll 4
      for (uint32_t k = 0; k < nc; ++k) {
        const float4 pj = P[base + k + gshift];
        const uint32_t bit = (b2_pred(pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, R2) ? 1u : 0u) << k;
        m |= bit;
        if (!STORE_BCE) mf |= tag_is_bce(tag_of(U[base + k + gshift].w)) ? 0u : bit;
      }
    }
    uint32_t valid = nc >= 32 ? 0xffffffffu : ((1u << nc) - 1u);
    if (base < ob) valid &= ~((1u << (ob - base)) - 1u);   // the aligned chunk's slots before ob
    if (self - base < nc) valid &= ~(1u << (self - base));
    m &= valid;
    cnt += __popc(m);
    const uint32_t s = STORE_BCE ? m : (mf & valid);
    if (s) {
      if (nw == FMW) {   // this thread's mask slots are full: append what they hold now
        drain_masks<STAGED>(sm, nw, nent, w);
        nw = 0;
        nent = 0;
      }
      sm.mw[nw][threadIdx.x] = s;
      sm.wb[nw][threadIdx.x] = (uint16_t)base;
      ++nw;
      nent += __popc(s);
    }
  }
}

// the 9 candidate runs of particle i (window offset self, column q, cell z = cz); returns |P(i)|
template <bool STAGED, bool STORE_BCE>
__device__ __forceinline__ uint32_t filter_particle(float R2, FilterSmem& sm, const float4* __restrict__ P,
                                                    const float4* __restrict__ U, int q, int cz, uint32_t self,
                                                    float4 pi, ListWriter& w) {
  int nw = 0;
  uint32_t nent = 0;
  // (measured: pruning neighbour cells by their box distance removes ~24 % of the candidates
  //  but costs more in divergence than it saves; the full 27-cell stencil is kept)
  uint32_t cnt = 0;
#pragma unroll 1
  for (int da = -1; da <= 1; ++da) {
#pragma unroll 1
    for (int db = -1; db <= 1; ++db) {
      uint32_t ob, oe;
      int r;
      cand_range(sm, q, da, db, cz, ob, oe, r);
      const uint32_t gshift = sm.run_start[r] - sm.run_base[r];
      // the own run holds i itself: its bit is masked off (j != i, A18)
      filter_range<STAGED, STORE_BCE>(R2, sm, P, U, ob, oe, (da == 0 && db == 0) ? self : ~0u, gshift, pi, cnt, nw,
                                      nent, w);
    }
  }
  drain_masks<STAGED>(sm, nw, nent, w);
  return cnt;
}

template <bool STAGED>
__device__ __forceinline__ int filter_tile(const Grid& g, FilterSmem& sm, const float4* __restrict__ P,
                                            const float4* __restrict__ U, uint16_t* __restrict__ list,
                                            uint32_t* __restrict__ nlist, uint32_t* __restrict__ count_all,
                                            const uint32_t* __restrict__ cell_of, ListShape ls, int store_all,
                                            ErrLatch* err, const uint32_t* __restrict__ ids, long long step) {
  const uint32_t n_i = sm.col_pref[NCOL];
  int has_marker = 0;
  for (uint32_t t = threadIdx.x; t < n_i; t += blockDim.x) {
    int q;
    const uint32_t i = tile_particle(sm, t, q);
    const int r_self = (1 + q / TY) * WRY + (1 + q % TY);
    const uint32_t self = sm.run_base[r_self] + (i - sm.run_start[r_self]);
    const int cz = (int)(cell_of[i] % (uint32_t)g.dims[2]);
    const float4 pi = STAGED ? make_float4(sm.X[self], sm.Y[self], sm.Z[self], 0.f) : P[i];
    const bool bce = tag_is_bce(tag_of(U[i].w));
    has_marker |= bce ? 1 : 0;
    if (bce) {
      atomicMin(const_cast<int*>(&sm.mzmin), cz);
      atomicMax(const_cast<int*>(&sm.mzmax), cz);
    }
    const bool fluid_only = !store_all && bce;
    ListWriter w;
    w.init(list, i, ls);
    const uint32_t cnt = fluid_only ? filter_particle<STAGED, false>(g.R2, sm, P, U, q, cz, self, pi, w)
                                    : filter_particle<STAGED, true>(g.R2, sm, P, U, q, cz, self, pi, w);
    w.flush(STAGED ? self << 4 : self);
    nlist[i] = (uint32_t)min(w.k, ls.cap);
    count_all[i] = cnt;
    if (w.k > ls.cap) latch_error(err, -9 /*CRM_E_CAPACITY*/, (long long)ids[i], step, (long long)w.k);
  }
  return has_marker;
}

// 128 threads x 5 CTAs per SM (shared memory: the window's positions + the threads' mask slots)
__global__ void __launch_bounds__(FILTER_THREADS, CRM_FILTER_MINB)
    k_filter_t(Grid g, const uint32_t* __restrict__ cell_start, const float4* __restrict__ P,
               const float4* __restrict__ U, uint16_t* __restrict__ list, uint32_t* __restrict__ nlist,
               uint32_t* __restrict__ count_all, const uint32_t* __restrict__ cell_of, ListShape ls, int store_all,
               ErrLatch* err, const uint32_t* __restrict__ ids, long long step, long long tile_base,
               const uint32_t* __restrict__ tile_list, uint32_t* __restrict__ mtiles, uint32_t* __restrict__ mcount) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FilterSmem& sm = *reinterpret_cast<FilterSmem*>(smem_raw);
  if (latched(err)) return;
  const long long tile = tile_list ? (long long)tile_list[blockIdx.x] : tile_base + (long long)blockIdx.x;
  const TileGeom G = tile_geom(g, tile);
  tile_setup(g, G, cell_start, sm);
  if (sm.col_pref[NCOL] == 0) return;
  if (sm.run_base[WR] > 65535u) {   // 16-bit list entries
    if (threadIdx.x == 0) latch_error(err, -9, -1, step, (long long)sm.run_base[WR]);
    return;
  }
  filter_stage(P, U, sm);
  if (threadIdx.x == 0) {
    sm.mzmin = 0x7fffffff;
    sm.mzmax = -1;
  }
  tile_stage_wait();
  __syncthreads();
  const int has = sm.staged ? filter_tile<true>(g, sm, P, U, list, nlist, count_all, cell_of, ls, store_all, err, ids, step)
                            : filter_tile<false>(g, sm, P, U, list, nlist, count_all, cell_of, ls, store_all, err, ids, step);
  // the tiles holding markers: the BCE kernels run over these only (any order: tiles are independent)
  // with the rows z0 + zl .. z0 + zh (0 <= zl <= zh < TZ) that hold them in bits 28-31 (tiles < 2^28)
  if (__syncthreads_or(has) && threadIdx.x == 0) {
    const uint32_t zl = (uint32_t)(sm.mzmin - G.z0) & 3u, zh = (uint32_t)(sm.mzmax - G.z0) & 3u;
    mtiles[atomicAdd(mcount, 1u)] = (uint32_t)tile | (zl << 28) | (zh << 30);
  }
}

}  // namespace crmk
