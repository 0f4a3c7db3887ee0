// filter.cuh — Alg. 1 neighbour lists in a kernel of their own.
//
//   k_filter_t  one CTA per cell tile; stages only the window's positions (16 B) and a BCE flag
//               (1 B) per particle — a quarter of the rates kernels' 56-B window — so several CTAs
//               share an SM and the branchy, latency-bound candidate sweep runs at high occupancy
//               instead of inside the register- and shared-memory-limited pair kernels.  Every
//               particle of the tile gets its list: fluid particles all neighbours, markers their
//               fluid neighbours (Adami sums run over fluid only), or all with store_all
//               (debug export; nlist = |P(i)| for the structure checks).  The tiles that hold
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
  // offset of each mask's bit 0 (group-major path: its byte offset, 16 x the slot, as the list entry
  // needs it); drained into the list once the particle's sweep is complete
  uint32_t mw[FMW][FILTER_THREADS];
  uint16_t wb[FMW][FILTER_THREADS];
  uint2 pmask[33];   // group-major path: gm_prefix_mask(x) for x = 0..32
};

// positions + tag words of the window (LDGSTS; the tags land in the mask slots and become the BCE
// flags after the wait)
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
      // the tag word too (into the mask slots, unused until the sweep): no synchronous load in the
      // staging loop (measured: k_filter 11.96 -> 11.77 ms against a load of U[gidx] per slot)
      __pipeline_memcpy_async(&sm.mw[0][0] + idx, reinterpret_cast<const float*>(&U[gidx]) + 3, sizeof(float));
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

// the same predicate as b2_group8, left in sign-byte form: bit 7 of byte p of wa (wb) = candidate p
// (4 + p) is a neighbour, every other bit 0
__device__ __forceinline__ void b2_group8_bytes(const FilterSmem& sm, uint32_t j, unsigned long long xi2,
                                                unsigned long long yi2, unsigned long long zi2,
                                                unsigned long long R2x2, uint32_t& wa, uint32_t& wb) {
  const ulonglong2 xa = *reinterpret_cast<const ulonglong2*>(&sm.X[j]);
  const ulonglong2 ya = *reinterpret_cast<const ulonglong2*>(&sm.Y[j]);
  const ulonglong2 za = *reinterpret_cast<const ulonglong2*>(&sm.Z[j]);
  const ulonglong2 xb = *reinterpret_cast<const ulonglong2*>(&sm.X[j + 4]);
  const ulonglong2 yb = *reinterpret_cast<const ulonglong2*>(&sm.Y[j + 4]);
  const ulonglong2 zb = *reinterpret_cast<const ulonglong2*>(&sm.Z[j + 4]);
  const unsigned long long d0 = b2_r2m(xa.x, ya.x, za.x, xi2, yi2, zi2, R2x2);
  const unsigned long long d1 = b2_r2m(xa.y, ya.y, za.y, xi2, yi2, zi2, R2x2);
  const unsigned long long d2 = b2_r2m(xb.x, yb.x, zb.x, xi2, yi2, zi2, R2x2);
  const unsigned long long d3 = b2_r2m(xb.y, yb.y, zb.y, xi2, yi2, zi2, R2x2);
  wa = __byte_perm(__byte_perm((uint32_t)d0, (uint32_t)(d0 >> 32), 0x0073),
                   __byte_perm((uint32_t)d1, (uint32_t)(d1 >> 32), 0x0073), 0x5410) & 0x80808080u;
  wb = __byte_perm(__byte_perm((uint32_t)d2, (uint32_t)(d2 >> 32), 0x0073),
                   __byte_perm((uint32_t)d3, (uint32_t)(d3 >> 32), 0x0073), 0x5410) & 0x80808080u;
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

// ---- bank-group-major list order (staged windows; CRM_LIST_ORDER != scan) ----------------------
// The pair kernels gather each entry's 16-B window slots; the 8 lanes of a quarter warp read their
// k-th entries at once, conflict-free only when the 8 slots lie in distinct bank groups (slot mod 8).
// Lists in candidate order put the lanes' groups at random (offline model of the C5 lists: 2.38
// shared-memory wavefronts per ideal one); a list that holds i's entries of group g0, then g0 + 1,
// ... (mod 8), each group in candidate order, with g0 = i's tile slot mod 8 (= its lane in the
// quarter), keeps the lanes of a quarter in distinct groups for most steps (1.62 in the model;
// measured k_rates_A/B 13.5/13.9 -> 11.7/12.3 ms).  To emit that order without buffering the list,
// the sweep stores its hits transposed: chunks of 32 candidates start on a multiple of 8, so the
// candidate at chunk offset 8n + p (n < 4) is in group p; its bit goes to bit n of byte p (the
// sign-byte form the predicate produces anyway), two chunks share a byte (nibbles), and the bytes
// of group g are collected in g's own words (4 bytes = 8 chunks per word, GMW words).  The drain
// then walks the 8 group strings in rotated order, one entry per iteration (lockstep appends).
constexpr int GMW = FMW / 8;   // words per group string: 8 GMW chunks per particle before an early drain

// transposed valid mask of the first x (0..32) candidates of a chunk: bit n of byte p (groups 0-3
// in .x, 4-7 in .y) for every candidate 8n + p < x
__device__ __forceinline__ uint2 gm_prefix_mask(uint32_t x) {
  uint32_t a = 0, b = 0;
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const uint32_t cnt = x > (uint32_t)p ? min(4u, (x - (uint32_t)p + 7u) >> 3) : 0u;   // n with 8n + p < x
    const uint32_t nib = (1u << cnt) - 1u;
    if (p < 4) a |= nib << (8 * p); else b |= nib << (8 * (p - 4));
  }
  return make_uint2(a, b);
}

struct GmState {
  uint32_t A, B;      // the open byte position (chunks 2p, 2p+1 as low/high nibbles; groups 0-3 / 4-7)
  int nch;            // chunks stored
  uint32_t nent;      // entries stored
};

__device__ __forceinline__ void gm_reset(GmState& st) {
  st.A = st.B = 0u;
  st.nch = 0;
  st.nent = 0;
}

// 4x4 byte transpose: out word k = byte k of r0, r1, r2, r3
__device__ __forceinline__ void bytes4x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  const uint32_t a = __byte_perm(r0, r1, 0x5140), b = __byte_perm(r0, r1, 0x7362);
  const uint32_t c = __byte_perm(r2, r3, 0x5140), d = __byte_perm(r2, r3, 0x7362);
  r0 = __byte_perm(a, c, 0x5410);
  r1 = __byte_perm(a, c, 0x7632);
  r2 = __byte_perm(b, d, 0x5410);
  r3 = __byte_perm(b, d, 0x7632);
}

// append the particle's stored entries in group-major order and reset the state.  Stored so far:
// per byte position p (two chunks) the words (A, B) at mw[2p], mw[2p + 1]; transposed in place, 4
// byte positions at a time, into group words: mw[8 wd + g] = bytes 4 wd .. 4 wd + 3 of group g.
__device__ __forceinline__ void gm_drain(FilterSmem& sm, GmState& st, uint32_t g0, ListWriter& w, uint32_t fill,
                                         bool final) {
  const uint32_t t = threadIdx.x;
  const int nb = (st.nch + 1) >> 1;   // byte positions
  uint32_t NZ = 0;                    // bit 4 g + wd: group g's word wd holds entries
  for (int wd = 0; 4 * wd < nb; ++wd) {
    uint32_t r[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool in = 4 * wd + k < nb;
      r[k] = in ? sm.mw[8 * wd + 2 * k][t] : 0u;       // groups 0-3 of byte position 4 wd + k
      r[4 + k] = in ? sm.mw[8 * wd + 2 * k + 1][t] : 0u;   // groups 4-7
    }
    bytes4x4(r[0], r[1], r[2], r[3]);
    bytes4x4(r[4], r[5], r[6], r[7]);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      sm.mw[8 * wd + g][t] = r[g];
      NZ |= (r[g] ? 1u : 0u) << (4 * g + wd);
    }
  }
  // the non-empty words in emission order (groups g0, g0 + 1, ...): NZ rotated by 4 g0
  uint32_t nz = __funnelshift_r(NZ, NZ, 4u * (g0 & 7u));
  uint32_t W = 0, wd = 0, g = 0;
  // one entry: advance to the next non-empty word when W is spent (one ffs, no search, no branch:
  // the lanes of a warp reach the ends of their words at different entries), take its lowest bit
  auto next = [&]() -> uint32_t {
    // (the indices stay inside the mask slots after the last entry, when nz and W are 0: the padded
    //  tail of the last chunk calls this too)
    const bool adv = W == 0u;
    const uint32_t pos = (__ffs(nz) - 1) & 31u;
    nz = adv ? (nz & (nz - 1)) : nz;
    wd = adv ? min(pos & 3u, (uint32_t)GMW - 1u) : wd;
    g = adv ? ((g0 + (pos >> 2)) & 7u) : g;
    const uint32_t Wn = sm.mw[wd * 8 + g][t];
    W = adv ? Wn : W;
    const uint32_t q = (__ffs(W) - 1) & 31u;   // bit q: chunk 8 wd + (q >> 2), candidate 8 (q & 3) + g of it
    W &= W - 1;
    return sm.wb[8 * wd + (q >> 2)][t] + ((q & 3u) << 7) + (g << 4);   // wb holds 16 x the chunk base
  };
  if (final && w.k == 0 && (int)st.nent <= w.cap) {
    // the whole list at once (no early drain): whole chunks of 8 entries, one 16-B store each, the
    // last chunk padded with the particle's own slot; e = 8c + u is the same on every lane of a
    // warp, so the chunk's register positions are compile-time
    uint4* row = reinterpret_cast<uint4*>(w.cur);
    const uint32_t nchk = max(1u, (st.nent + 7u) >> 3);
    // whole chunks without the tail select, then the last (padded) chunk (with the pre-scaled chunk
    // bases: k_filter 13.15 -> 12.74 ms)
    for (uint32_t c = 0; c + 1 < nchk; ++c) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = next();
      row[(size_t)c * w.stride] = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16),
                                             v[6] | (v[7] << 16));
    }
    {
      const uint32_t c = nchk - 1;
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t x = next();
        v[u] = 8u * c + (uint32_t)u < st.nent ? x : fill;
      }
      row[(size_t)c * w.stride] = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16),
                                             v[6] | (v[7] << 16));
    }
    w.k = (int)st.nent;
    w.closed = true;
  } else {
    for (uint32_t e = 0; e < st.nent; ++e) w.push(next());
  }
  gm_reset(st);
}


// store one chunk's transposed hits (a, b: groups 0-3 / 4-7, bit n of byte p) at window base
__device__ __forceinline__ void gm_store_chunk(FilterSmem& sm, GmState& st, uint32_t a, uint32_t b, uint32_t base,
                                               uint32_t g0, ListWriter& w) {
  if (st.nch == FMW) gm_drain(sm, st, g0, w, 0u, false);   // all mask slots used: append what they hold now
  const uint32_t t = threadIdx.x;
  sm.wb[st.nch][t] = (uint16_t)(base << 4);   // staged windows: base < 4096
  st.nent += __popc(a) + __popc(b);
  {   // branch-free: the open byte position is stored with every chunk (the odd one completes it;
      // measured against a store per completed pair: k_filter 11.75 -> 11.45 ms)
    const bool odd = (st.nch & 1) != 0;
    const int p = st.nch >> 1;
    st.A = odd ? (st.A | (a << 4)) : a;
    st.B = odd ? (st.B | (b << 4)) : b;
    sm.mw[2 * p][t] = st.A;
    sm.mw[2 * p + 1][t] = st.B;
  }
  ++st.nch;
}

// Alg. 1 over one candidate range, staged window, group-major storage (see above)
// MODE 0: every neighbour stored (fluid particles, store_all); 1: fluid neighbours only (markers);
// 2: per lane, fonly selects 1 (a warp holding markers and fluid: one sweep with the flags instead of
// the two paths of a divergent warp)
template <int MODE>
__device__ __forceinline__ void filter_range_gm(float R2, FilterSmem& sm, uint32_t ob, uint32_t oe, uint32_t self,
                                                const float4& pi, GmState& st, uint32_t g0,
                                                ListWriter& w, bool fonly) {
  constexpr bool STORE_BCE = MODE == 0;
  const unsigned long long xi2 = f2_splat(pi.x), yi2 = f2_splat(pi.y), zi2 = f2_splat(pi.z);
  const unsigned long long R2x2 = f2_splat(R2);
  for (uint32_t base = ob & ~7u; base < oe; base += 32) {
    const uint32_t nc = min(32u, oe - base);
    uint32_t a = 0, b = 0, fa = 0, fb = 0;
#pragma unroll
    for (uint32_t n = 0; n < 4; ++n) {
      const uint32_t k8 = 8 * n;
      if (k8 >= nc) break;
      uint32_t wa, wb;
      b2_group8_bytes(sm, base + k8, xi2, yi2, zi2, R2x2, wa, wb);   // bit 7 of byte p: candidate p (wb: 4 + p)
      a |= wa >> (7u - n);
      b |= wb >> (7u - n);
      if (!STORE_BCE) {   // fluid candidates only: the flags are bytes 0/1
        const uint32_t f0 = *reinterpret_cast<const uint32_t*>(&sm.bce[base + k8]);
        const uint32_t f1 = *reinterpret_cast<const uint32_t*>(&sm.bce[base + k8 + 4]);
        fa |= (wa & ~(f0 << 7)) >> (7u - n);
        fb |= (wb & ~(f1 << 7)) >> (7u - n);
      }
    }
    // valid candidates [max(ob, base), min(oe, base + 32)) without i itself
    const uint2 vhi = sm.pmask[nc], vlo = sm.pmask[base < ob ? ob - base : 0u];
    uint32_t va = vhi.x & ~vlo.x, vb = vhi.y & ~vlo.y;
    if (self - base < nc) {
      const uint32_t o = self - base, bit = 1u << (8u * (o & 3u) + (o >> 3));
      if (o & 4u) vb &= ~bit; else va &= ~bit;
    }
    a &= va;
    b &= vb;
    if (MODE == 1 || (MODE == 2 && fonly)) {
      a = fa & va;
      b = fb & vb;
    }
    gm_store_chunk(sm, st, a, b, base, g0, w);   // empty chunks too (no divergent store: -0.12 ms)
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
                                             uint32_t gshift, const float4& pi, int& nw,
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
template <bool STAGED, bool STORE_BCE, int MODE = STORE_BCE ? 0 : 1>
__device__ __forceinline__ void filter_particle(float R2, FilterSmem& sm, const float4* __restrict__ P,
                                                    const float4* __restrict__ U, int q, int cz, uint32_t self,
                                                    float4 pi, ListWriter& w, bool gmaj, uint32_t g0,
                                                    bool fonly = false) {
  int nw = 0;
  uint32_t nent = 0;
  GmState st;
  if (STAGED && gmaj) gm_reset(st);
  // (measured: pruning neighbour cells by their box distance removes ~24 % of the candidates
  //  but costs more in divergence than it saves; the full 27-cell stencil is kept)
#pragma unroll 1
  for (int da = -1; da <= 1; ++da) {
#pragma unroll 1
    for (int db = -1; db <= 1; ++db) {
      uint32_t ob, oe;
      int r;
      cand_range(sm, q, da, db, cz, ob, oe, r);
      const uint32_t gshift = sm.run_start[r] - sm.run_base[r];
      // the own run holds i itself: its bit is masked off (j != i, A18)
      const uint32_t sf = (da == 0 && db == 0) ? self : ~0u;
      if (STAGED && gmaj) filter_range_gm<MODE>(R2, sm, ob, oe, sf, pi, st, g0, w, fonly);
      else filter_range<STAGED, STORE_BCE>(R2, sm, P, U, ob, oe, sf, gshift, pi, nw, nent, w);
    }
  }
  if (STAGED && gmaj) gm_drain(sm, st, g0, w, self << 4, true);
  else drain_masks<STAGED>(sm, nw, nent, w);
}

template <bool STAGED>
__device__ __forceinline__ int filter_tile(const Grid& g, FilterSmem& sm, const float4* __restrict__ P,
                                            const float4* __restrict__ U, uint16_t* __restrict__ list,
                                            uint32_t* __restrict__ nlist,
                                            const uint32_t* __restrict__ cell_of, ListShape ls, int store_all,
                                            ErrLatch* err, const uint32_t* __restrict__ ids, long long step,
                                            bool gmaj) {
  const uint32_t n_i = sm.col_pref[NCOL];
  int has_marker = 0;
  for (uint32_t t = threadIdx.x; t < n_i; t += blockDim.x) {
    int q;
    const uint32_t i = tile_particle(sm, t, q);
    const int r_self = (1 + q / TY) * WRY + (1 + q % TY);
    const uint32_t self = sm.run_base[r_self] + (i - sm.run_start[r_self]);
    // the particle's cell row and kind from the tile geometry and the staged window (no global
    // loads on the per-particle path when staged): cz = the cell of the own run holding slot i
    int cz;
    bool bce;
    if (STAGED) {
      int k = 0;
#pragma unroll
      for (int kk = 1; kk < TZ + 2; ++kk) k += (kk <= sm.zhi - sm.zlo && sm.wcs[r_self][kk] <= i) ? 1 : 0;
      cz = sm.zlo + k;
      bce = sm.bce[self] != 0;
    } else {
      cz = (int)(cell_of[i] % (uint32_t)g.dims[2]);
      bce = tag_is_bce(tag_of(U[i].w));
    }
    const float4 pi = STAGED ? make_float4(sm.X[self], sm.Y[self], sm.Z[self], 0.f) : P[i];
    has_marker |= bce ? 1 : 0;
    if (bce) {
      atomicMin(const_cast<int*>(&sm.mzmin), cz);
      atomicMax(const_cast<int*>(&sm.mzmax), cz);
    }
    const bool fluid_only = !store_all && bce;
    ListWriter w;
    w.init(list, i, ls);
    // a warp's lanes are one kind (one sweep, no flags for fluid) or mixed (one sweep with the flags:
    // a divergent warp would run both sweeps; measured k_filter 12.71 -> 12.05 ms on the C5 bed)
    const unsigned am = __activemask();
    const bool any_f = __any_sync(am, fluid_only), all_f = __all_sync(am, fluid_only);
    if (STAGED && gmaj && any_f && !all_f)
      filter_particle<STAGED, false, 2>(g.R2, sm, P, U, q, cz, self, pi, w, gmaj, t & 7u, fluid_only);
    else if (fluid_only)
      filter_particle<STAGED, false>(g.R2, sm, P, U, q, cz, self, pi, w, gmaj, t & 7u);
    else
      filter_particle<STAGED, true>(g.R2, sm, P, U, q, cz, self, pi, w, gmaj, t & 7u);
    w.flush(STAGED ? self << 4 : self);
    nlist[i] = (uint32_t)min(w.k, ls.cap);
    if (w.k > ls.cap) latch_error(err, -9 /*CRM_E_CAPACITY*/, (long long)ids[i], step, (long long)w.k);
  }
  return has_marker;
}

// 128 threads x 5 CTAs per SM (shared memory: the window's positions + the threads' mask slots)
__global__ void __launch_bounds__(FILTER_THREADS, CRM_FILTER_MINB)
    k_filter_t(Grid g, const uint32_t* __restrict__ cell_start, const float4* __restrict__ P,
               const float4* __restrict__ U, uint16_t* __restrict__ list, uint32_t* __restrict__ nlist,
               const uint32_t* __restrict__ cell_of, ListShape ls, int store_all,
               ErrLatch* err, const uint32_t* __restrict__ ids, long long step, long long tile_base,
               const uint32_t* __restrict__ tile_list, uint32_t* __restrict__ mtiles, uint32_t* __restrict__ mcount,
               int order) {
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
  if (threadIdx.x < 33) sm.pmask[threadIdx.x] = gm_prefix_mask(threadIdx.x);
  if (threadIdx.x == 0) {
    sm.mzmin = 0x7fffffff;
    sm.mzmax = -1;
  }
  tile_stage_wait();
  __syncthreads();
  if (sm.staged) {
    for (uint32_t idx = threadIdx.x; idx < sm.run_base[WR]; idx += blockDim.x)
      sm.bce[idx] = tag_is_bce((&sm.mw[0][0])[idx]) ? 1 : 0;
    __syncthreads();
  }
  const bool gmaj = order == 1;
  const int has = sm.staged ? filter_tile<true>(g, sm, P, U, list, nlist, cell_of, ls, store_all, err, ids, step, gmaj)
                            : filter_tile<false>(g, sm, P, U, list, nlist, cell_of, ls, store_all, err, ids, step, gmaj);
  // the tiles holding markers: the BCE kernels run over these only (any order: tiles are independent)
  // with the rows z0 + zl .. z0 + zh (0 <= zl <= zh < TZ) that hold them in bits 28-31 (tiles < 2^28)
  if (__syncthreads_or(has) && threadIdx.x == 0) {
    const uint32_t zl = (uint32_t)(sm.mzmin - G.z0) & 3u, zh = (uint32_t)(sm.mzmax - G.z0) & 3u;
    mtiles[atomicAdd(mcount, 1u)] = (uint32_t)tile | (zl << 28) | (zh << 30);
  }
}

}  // namespace crmk
