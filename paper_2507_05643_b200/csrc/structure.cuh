// structure.cuh — cell binning, deterministic counting sort by (cell, id), reorder and
// neighbour lists (§4.1; rules B1–B5 of DESIGN.md).
//
// Per step (ps_freq = 1):
//   k_bin        hash every particle, count per cell (atomics), remember arrival rank
//   scan         exclusive scan of the counts -> cellStart (CSR, M+1)
//   k_scatter    slot = cellStart[c] + arrival  (arrival order is not deterministic)
//   k_reorder    rank inside the cell by id -> final (cell, id) position; moves the
//                56-B state with float4/float2 vector loads/stores
// The Alg. 1 filter itself runs inside the tiled kernels (tiled.cuh), fused with the pair loops.
#pragma once
#include "common.cuh"

namespace crmk {

// ---------------------------------------------------------------------------------------
// B1: cell coordinate = floor((x - lo) / s), IEEE fp32 sub + div (no reciprocal multiply)
__device__ __forceinline__ float b1_floor(float x, float lo, float s) {
  return floorf(__fdiv_rn(__fsub_rn(x, lo), s));
}

// B2: dx = xj - xi; r2 = fma(dz,dz, fma(dy,dy, dx*dx)); neighbour iff r2 < R2
__device__ __forceinline__ bool b2_pred(float xi, float yi, float zi, float xj, float yj, float zj, float R2) {
  const float dx = __fsub_rn(xj, xi);
  const float dy = __fsub_rn(yj, yi);
  const float dz = __fsub_rn(zj, zi);
  const float r2 = __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
  return r2 < R2;
}

// ---------------------------------------------------------------------------------------
// moving markers: x = p + R x_local at the pose of the step start (body 0 never moves)
__global__ void k_markers_place(int nm, const uint32_t* __restrict__ moving_ids,
                                const float4* __restrict__ xlocal, const uint32_t* __restrict__ slot_of_id,
                                const Pose* __restrict__ pose, float4* __restrict__ P, float4* __restrict__ L,
                                float4* __restrict__ U) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nm) return;
  const uint32_t id = moving_ids[k];
  const uint32_t s = slot_of_id[id];
  if (s == 0xffffffffu) return;   // multi-GPU: the marker lives on another slab
  const uint32_t b = tag_body(tag_of(U[s].w));
  const float4 xl = xlocal[k];
  const Pose& q = pose[b];
  float4 p = P[s];
  p.x = q.pos[0] + q.R[0] * xl.x + q.R[1] * xl.y + q.R[2] * xl.z;
  p.y = q.pos[1] + q.R[3] * xl.x + q.R[4] * xl.y + q.R[5] * xl.z;
  p.z = q.pos[2] + q.R[6] * xl.x + q.R[7] * xl.y + q.R[8] * xl.z;
  P[s] = p;
  L[s] = make_float4(0.f, 0.f, 0.f, 0.f);   // placed from the pose: no compensation term
  U[s].w = __uint_as_float(tag_of(U[s].w) & TAG_FLAGS);
}

// hash + per-cell count; the error latch reports particles outside the grid.
// Particles whose tag has a bit of drop_mask (multi-GPU ghosts / emigrants) get the sentinel key
// M: they sort behind every cell and are not kept.
// Inactive particles of Alg. 3 (act[i] == 2, act may be NULL) get the sentinel key too; k_reorder
// keeps them (keep_tail) behind the active set instead of dropping them.
__global__ void k_bin(int n, const float4* __restrict__ P, const float4* __restrict__ U,
                      const uint32_t* __restrict__ ids, Grid g, uint32_t drop_mask, const uint8_t* __restrict__ act,
                      uint32_t* __restrict__ key, uint32_t* __restrict__ arrival, uint32_t* __restrict__ cell_count,
                      ErrLatch* err, long long step, const uint32_t* __restrict__ dn) {
  if (dn) n = (int)*dn;   // slabs: the local count lives on the device (grid over the capacity)
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  uint32_t c = g.M;
  if (valid && !((drop_mask && (tag_of(U[i].w) & drop_mask)) || (act && act[i] == 2))) {
    const float4 p = P[i];
    float f[3] = {b1_floor(p.x, g.lo[0], g.s), b1_floor(p.y, g.lo[1], g.s), b1_floor(p.z, g.lo[2], g.s)};
    int c3[3];
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const bool in = (f[a] >= 0.0f) && (f[a] < (float)g.dims[a]);   // false for NaN too
      ok = ok && in;
      c3[a] = in ? (int)f[a] : 0;
    }
    if (!ok) latch_error(err, -2 /*CRM_E_DOMAIN*/, (long long)ids[i], step, 0);
    c = (uint32_t)c3[0] * (uint32_t)(g.dims[1] * g.dims[2]) + (uint32_t)c3[1] * (uint32_t)g.dims[2] + (uint32_t)c3[2];
  }
  // arrival rank inside the cell: one atomic per distinct cell of the warp (the input is in the
  // previous step's cell order, so a warp covers few cells); only a temporary slot — the final
  // order inside a cell is by id (k_reorder)
  const unsigned vm = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const int lane = threadIdx.x & 31;
  const unsigned peers = __match_any_sync(vm, c);
  const int leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(&cell_count[c], (uint32_t)__popc(peers));
  base = __shfl_sync(peers, base, leader);
  key[i] = c;
  arrival[i] = base + (uint32_t)__popc(peers & ((1u << lane) - 1u));
}

// ---------------------------------------------------------------------------------------
// exclusive scan of uint32 (tiles of SCAN_BS * SCAN_IPT), recursive over tile sums
constexpr int SCAN_BS = 512;
constexpr int SCAN_IPT = 8;
constexpr int SCAN_TILE = SCAN_BS * SCAN_IPT;

__global__ void __launch_bounds__(SCAN_BS) k_scan_tiles(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                        uint32_t* __restrict__ tile_sums, long long n) {
  __shared__ uint32_t warp_sums[SCAN_BS / 32];
  const long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_IPT;
  uint32_t v[SCAN_IPT];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    v[k] = (base + k < n) ? in[base + k] : 0u;
    sum += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = (lane < SCAN_BS / 32) ? warp_sums[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < SCAN_BS / 32) warp_sums[lane] = wi - w;   // exclusive warp offsets
    if (lane == SCAN_BS / 32 - 1) tile_sums[blockIdx.x] = wi;
  }
  __syncthreads();
  uint32_t run = warp_sums[warp] + incl - sum;
#pragma unroll
  for (int k = 0; k < SCAN_IPT; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

__global__ void k_scan_add(uint32_t* __restrict__ out, const uint32_t* __restrict__ tile_off, long long n) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += tile_off[i / SCAN_TILE];
}

__global__ void k_copy_u32(uint32_t* dst, const uint32_t* src) { *dst = *src; }

// ---------------------------------------------------------------------------------------
// Slab rebuild, one pass over the local particles (replaces a first sort): last step's ghosts are
// marked dropped; an owned particle now in the neighbour's first plane is an emigrant — its state goes
// to that neighbour (segment E of the pack buffer of that side) and this rank keeps it as a ghost;
// an owned particle in this slab's first / last plane is copied to the left / right pack buffer
// (segment G: the neighbour's ghost plane).  Order inside a segment is arbitrary: the receiver sorts
// by (cell, id).  A particle that crossed more than one plane latches CRM_E_DOMAIN (aux 1).
struct SlabPack {
  float4 *P[2], *L[2], *U[2], *S1[2];
  float2* S2[2];
  uint32_t* id[2];
  uint32_t* cnt;      // [E_left, G_left, E_right, G_right]
  uint32_t cap_e, cap_g;
};
__device__ __forceinline__ void slab_put(const SlabPack& pk, int d, uint32_t slot, const float4& p, const float4& l,
                                         const float4& u, const float4& s1, const float2& s2, uint32_t id) {
  pk.P[d][slot] = p; pk.L[d][slot] = l; pk.U[d][slot] = u; pk.S1[d][slot] = s1; pk.S2[d][slot] = s2;
  pk.id[d][slot] = id;
}
__device__ __forceinline__ void slab_pack_one(int i, const float4* __restrict__ P, const float4* __restrict__ L,
                                              float4* __restrict__ U, const float4* __restrict__ S1,
                                              const float2* __restrict__ S2, const uint32_t* __restrict__ ids,
                                              const Grid& g, int x_lo, int x_hi, int has_l, int has_r,
                                              const SlabPack& pk, ErrLatch* err, long long step);
__global__ void k_slab_pack(int n, const float4* __restrict__ P, const float4* __restrict__ L, float4* __restrict__ U,
                            const float4* __restrict__ S1, const float2* __restrict__ S2,
                            const uint32_t* __restrict__ ids, Grid g, int x_lo, int x_hi, int has_l, int has_r,
                            SlabPack pk, ErrLatch* err, long long step, const uint32_t* __restrict__ dn) {
  n = (int)*dn;   // the local count (device word: the slab step has no host reads)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    slab_pack_one(i, P, L, U, S1, S2, ids, g, x_lo, x_hi, has_l, has_r, pk, err, step);
}
__device__ __forceinline__ void slab_pack_one(int i, const float4* __restrict__ P, const float4* __restrict__ L,
                                              float4* __restrict__ U, const float4* __restrict__ S1,
                                              const float2* __restrict__ S2, const uint32_t* __restrict__ ids,
                                              const Grid& g, int x_lo, int x_hi, int has_l, int has_r,
                                              const SlabPack& pk, ErrLatch* err, long long step) {
  const float4 u = U[i];
  const uint32_t tag = tag_of(u.w);
  if (tag & TAG_GHOST) {   // last step's ghost: leaves at this rebuild
    U[i].w = __uint_as_float(tag | TAG_DROP);
    return;
  }
  const float4 p = P[i];
  const int pl = (int)b1_floor(p.x, g.lo[0], g.s);
  const bool emi_l = pl < x_lo, emi_r = pl >= x_hi;
  if ((emi_l && (pl != x_lo - 1 || !has_l)) || (emi_r && (pl != x_hi || !has_r))) {
    latch_error(err, -2 /*CRM_E_DOMAIN*/, (long long)ids[i], step, 1);
    return;
  }
  const bool g_l = has_l && pl == x_lo, g_r = has_r && pl == x_hi - 1;
  if (!(emi_l || emi_r || g_l || g_r)) return;
  const float4 l = L[i], s1 = S1[i];
  const float2 s2 = S2[i];
  const uint32_t id = ids[i];
  if (emi_l || emi_r) {
    const int d = emi_l ? 0 : 1;
    const uint32_t k = atomicAdd(&pk.cnt[2 * d], 1u);
    if (k < pk.cap_e) slab_put(pk, d, k, p, l, u, s1, s2, id);
    else latch_error(err, -9 /*CRM_E_CAPACITY*/, (long long)id, step, 2);
    U[i].w = __uint_as_float(tag | TAG_GHOST);   // kept here as a ghost of the neighbour's first plane
    return;
  }
  if (g_l) {
    const uint32_t k = atomicAdd(&pk.cnt[1], 1u);
    if (k < pk.cap_g) slab_put(pk, 0, pk.cap_e + k, p, l, u, s1, s2, id);
    else latch_error(err, -9 /*CRM_E_CAPACITY*/, (long long)id, step, 2);
  }
  if (g_r) {
    const uint32_t k = atomicAdd(&pk.cnt[3], 1u);
    if (k < pk.cap_g) slab_put(pk, 1, pk.cap_e + k, p, l, u, s1, s2, id);
    else latch_error(err, -9 /*CRM_E_CAPACITY*/, (long long)id, step, 2);
  }
}

// Slab rebuild, receiver side.  The neighbours' pack buffers arrive whole (fixed capacity: the
// transfer sizes do not depend on device counts, so the step needs no host read and can be
// captured in a CUDA graph) with their counts in rv.cnt = [E, G from the left, E, G from the right].
// k_slab_counts (one thread) places the four segments behind the n local particles (d_slab[0] = n;
// d_slab[1..4] = segment starts; d_slab[0] becomes the new count) or latches CRM_E_CAPACITY;
// k_slab_append (gridDim.y = side) copies them: immigrants (E) must sit in this slab's boundary
// plane (a particle crosses at most one 2h plane per step), ghosts (G) get TAG_GHOST.
__global__ void k_slab_counts(uint32_t* __restrict__ d_slab, const uint32_t* __restrict__ rcnt, int has_l, int has_r,
                              uint32_t cap_e, uint32_t cap_g, uint32_t ncap, ErrLatch* err, long long step) {
  const uint32_t n = d_slab[0];
  const uint32_t el = has_l ? rcnt[0] : 0u, gl = has_l ? rcnt[1] : 0u;
  const uint32_t er = has_r ? rcnt[2] : 0u, gr = has_r ? rcnt[3] : 0u;
  if (el > cap_e || er > cap_e || gl > cap_g || gr > cap_g || (unsigned long long)n + el + gl + er + gr > ncap) {
    latch_error(err, -9 /*CRM_E_CAPACITY*/, -1, step, 3);
    d_slab[1] = d_slab[2] = d_slab[3] = d_slab[4] = n;   // nothing appended
    d_slab[5] = d_slab[6] = d_slab[7] = d_slab[8] = 0;
    return;
  }
  d_slab[1] = n; d_slab[2] = n + el; d_slab[3] = n + el + gl; d_slab[4] = n + el + gl + er;
  d_slab[5] = el; d_slab[6] = gl; d_slab[7] = er; d_slab[8] = gr;
  d_slab[0] = n + el + gl + er + gr;
}
__global__ void k_slab_append(const uint32_t* __restrict__ d_slab, SlabPack rv, float4* __restrict__ P,
                              float4* __restrict__ L, float4* __restrict__ U, float4* __restrict__ S1,
                              float2* __restrict__ S2, uint32_t* __restrict__ ids, Grid g, int x_lo, int x_hi,
                              ErrLatch* err, long long step) {
  if (latched(err)) return;
  const int d = blockIdx.y;   // 0: from the left neighbour, 1: from the right
  const uint32_t ne = d_slab[5 + 2 * d], ng = d_slab[6 + 2 * d];
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < ne + ng; j += gridDim.x * blockDim.x) {
    const bool emi = j < ne;
    const uint32_t k = emi ? j : rv.cap_e + (j - ne);                          // source slot
    const uint32_t dst = emi ? d_slab[1 + 2 * d] + j : d_slab[2 + 2 * d] + (j - ne);
    const float4 p = rv.P[d][k];
    float4 u = rv.U[d][k];
    const uint32_t id = rv.id[d][k];
    if (emi) {
      const float f = b1_floor(p.x, g.lo[0], g.s);
      if (!(f == (float)(d == 0 ? x_lo : x_hi - 1))) latch_error(err, -2 /*CRM_E_DOMAIN*/, (long long)id, step, 1);
    } else {
      u.w = __uint_as_float(tag_of(u.w) | TAG_GHOST);
    }
    P[dst] = p; L[dst] = rv.L[d][k]; U[dst] = u; S1[dst] = rv.S1[d][k]; S2[dst] = rv.S2[d][k];
    ids[dst] = id;
  }
}

// Per-stage halo of the slabs, fixed-capacity (graph-capturable): k_halo_pack copies this slab's
// boundary plane of side d = blockIdx.y (the cells [c0[d], c1[d]) — slots from cellStart) into the
// pack buffer of that side and its count into cnt[d]; k_halo_unpack copies the neighbour's plane
// into the ghost plane of side d (cells [c0[d], c1[d])), flags it TAG_GHOST and checks the counts
// agree (both sides hold the same particles in the same (cell, id) order).
struct HaloSide {
  uint32_t c0[2], c1[2];   // cell range per side
  int on[2];               // side has a neighbour
};
__global__ void k_halo_pack(const uint32_t* __restrict__ cell_start, HaloSide hs, const float4* __restrict__ P,
                            const float4* __restrict__ L, const float4* __restrict__ U, const float4* __restrict__ S1,
                            const float2* __restrict__ S2, SlabPack pk, uint32_t* __restrict__ cnt, ErrLatch* err,
                            long long step) {
  if (latched(err)) return;
  const int d = blockIdx.y;
  if (!hs.on[d]) return;
  const uint32_t b = cell_start[hs.c0[d]], n = cell_start[hs.c1[d]] - b;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    cnt[d] = n;
    if (n > pk.cap_g) latch_error(err, -9 /*CRM_E_CAPACITY*/, -1, step, 4);
  }
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < min(n, pk.cap_g); k += gridDim.x * blockDim.x) {
    pk.P[d][k] = P[b + k]; pk.L[d][k] = L[b + k]; pk.U[d][k] = U[b + k]; pk.S1[d][k] = S1[b + k];
    pk.S2[d][k] = S2[b + k];
  }
}
__global__ void k_halo_unpack(const uint32_t* __restrict__ cell_start, HaloSide hs, SlabPack rv,
                              const uint32_t* __restrict__ cnt, float4* __restrict__ P, float4* __restrict__ L,
                              float4* __restrict__ U, float4* __restrict__ S1, float2* __restrict__ S2, ErrLatch* err,
                              long long step) {
  if (latched(err)) return;
  const int d = blockIdx.y;
  if (!hs.on[d]) return;
  const uint32_t b = cell_start[hs.c0[d]], n = cell_start[hs.c1[d]] - b;
  if (blockIdx.x == 0 && threadIdx.x == 0 && cnt[d] != n) latch_error(err, -8 /*CRM_E_COMM*/, -1, step, (long long)cnt[d]);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < min(n, rv.cap_g); k += gridDim.x * blockDim.x) {
    float4 u = rv.U[d][k];
    u.w = __uint_as_float(tag_of(u.w) | TAG_GHOST);
    P[b + k] = rv.P[d][k]; L[b + k] = rv.L[d][k]; U[b + k] = u; S1[b + k] = rv.S1[d][k]; S2[b + k] = rv.S2[d][k];
  }
}

// slot_of_id entries of the particles of the old sorted set: invalid before the reorder writes the new
// set (O(local) instead of a fill over every id of the global input)
__global__ void k_clear_slots(int n, const uint32_t* __restrict__ ids, uint32_t* __restrict__ slot_of_id,
                              const uint32_t* __restrict__ dn) {
  if (dn) n = (int)*dn;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) slot_of_id[ids[i]] = 0xffffffffu;
}

// sum of |P(i)| over owned fluid particles (the directed pairs of the rates loops)
__global__ void k_pair_count(int n, const float4* __restrict__ U, const uint32_t* __restrict__ nlist,
                             unsigned long long* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (i < n) {
    const uint32_t t = tag_of(U[i].w);
    if (!tag_is_bce(t) && !tag_ghost(t)) v = nlist[i];   // a fluid list holds all of P(i)
  }
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

// Alg. 1 candidates: per particle, the particles of the 27 cells around its cell minus itself
// (out[0] over owned fluid particles, out[1] over markers) — the filter's algorithmic work
__global__ void k_candidate_count(int n, Grid g, const float4* __restrict__ U, const uint32_t* __restrict__ cell_of,
                                  const uint32_t* __restrict__ cell_start, unsigned long long* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long vf = 0, vb = 0;
  if (i < n) {
    const uint32_t t = tag_of(U[i].w);
    const uint32_t c = cell_of[i];
    if (!tag_ghost(t) && c < g.M) {
      const int Nz = g.dims[2], Ny = g.dims[1];
      const int cz = (int)(c % (uint32_t)Nz), cy = (int)((c / (uint32_t)Nz) % (uint32_t)Ny);
      const int cx = (int)(c / (uint32_t)(Ny * Nz));
      unsigned long long k = 0;
      for (int a = -1; a <= 1; ++a)
        for (int b = -1; b <= 1; ++b) {
          const int x = cx + a, y = cy + b;
          if (x < 0 || x >= g.dims[0] || y < 0 || y >= Ny) continue;
          const int z0 = max(cz - 1, 0), z1 = min(cz + 1, Nz - 1);
          const uint32_t c0 = (uint32_t)x * (uint32_t)(Ny * Nz) + (uint32_t)y * (uint32_t)Nz;
          k += cell_start[c0 + z1 + 1] - cell_start[c0 + z0];
        }
      (tag_is_bce(t) ? vb : vf) = k - 1;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    vf += __shfl_down_sync(0xffffffffu, vf, o);
    vb += __shfl_down_sync(0xffffffffu, vb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (vf) atomicAdd(&out[0], vf);
    if (vb) atomicAdd(&out[1], vb);
  }
}

__global__ void k_fill_u32(uint32_t* __restrict__ p, long long n, uint32_t v) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// ---------------------------------------------------------------------------------------
__global__ void k_scatter(int n, const uint32_t* __restrict__ key, const uint32_t* __restrict__ arrival,
                          const uint32_t* __restrict__ cell_start, const uint32_t* __restrict__ ids,
                          uint32_t* __restrict__ tmp_src, uint32_t* __restrict__ tmp_id, const uint32_t* __restrict__ dn) {
  if (dn) n = (int)*dn;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t slot = cell_start[key[i]] + arrival[i];
  tmp_src[slot] = (uint32_t)i;
  tmp_id[slot] = ids[i];
}

// final position = cellStart[c] + #(ids in the cell smaller than mine)  (B4, history-free)
__global__ void k_reorder(int n, const uint32_t* __restrict__ tmp_src, const uint32_t* __restrict__ tmp_id,
                          const uint32_t* __restrict__ key, const uint32_t* __restrict__ cell_start,
                          const float4* __restrict__ P, const float4* __restrict__ L,
                          const float4* __restrict__ U, const float4* __restrict__ S1,
                          const float2* __restrict__ S2, float4* __restrict__ Pn, float4* __restrict__ Ln,
                          float4* __restrict__ Un, float4* __restrict__ S1n, float2* __restrict__ S2n,
                          uint32_t* __restrict__ ids_n, uint32_t* __restrict__ cell_of,
                          uint32_t* __restrict__ slot_of_id, uint32_t M, int keep_tail, const uint32_t* __restrict__ dn) {
  if (dn) n = (int)*dn;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t i = tmp_src[s];
  const uint32_t myid = tmp_id[s];
  const uint32_t c = key[i];
  uint32_t d;
  if (c == M) {
    // multi-GPU: a ghost of the previous step or an emigrant, dropped; Alg. 3: an Inactive particle,
    // kept frozen behind the active set in its scatter slot (any order: it is nobody's neighbour)
    if (!keep_tail) return;
    d = (uint32_t)s;
  } else {
    const uint32_t b = cell_start[c], e = cell_start[c + 1];
    uint32_t rank = 0;
    for (uint32_t t = b; t < e; ++t) rank += (tmp_id[t] < myid) ? 1u : 0u;
    d = b + rank;
  }
  Pn[d] = P[i];
  Ln[d] = L[i];
  Un[d] = U[i];
  S1n[d] = S1[i];
  S2n[d] = S2[i];
  ids_n[d] = myid;
  cell_of[d] = c;
  slot_of_id[myid] = d;
}

}  // namespace crmk
