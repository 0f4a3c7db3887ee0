// tiled.cuh — the hot kernels: one CTA per cell tile, window staged in shared memory.
//
//   k_bce_t<0>   markers: Adami extrapolation at y_n           -> U, S of markers
//   k_rates_t<0> fluid: pair loop at y_n + y_mid = y_n + dt/2 f; markers
//                copied to the mid state
//   k_bce_t<1>   markers: extrapolation at y_mid with the stored lists
//   k_rates_t<1> fluid: pair loop at y_mid with the same lists (A17) + y_{n+1} = y_n + dt f
//                + mu(I) return map; moving-body markers: loads (A13)
// Each kernel: stage the window -> convert it to tile-relative compensated positions -> pair
// loops over the Alg. 1 lists of k_filter_t (filter.cuh) -> epilogue.
#pragma once
#include "common.cuh"
#include "physics.cuh"
#include "structure.cuh"
#include "tiles.cuh"

namespace crmk {

#ifdef CRM_EXP_TIMING
__device__ unsigned long long g_exp_timing[8192 * 6];   // timing experiment: per-CTA phase clocks
#endif

// ---------------------------------------------------------------------------------------
// neighbour state at list entry `e` (16 x window offset when staged, the offset in global mode); positions relative to the tile origin
// (see rel_pos), .w = rho_j (the BCE window keeps densities)
template <bool STAGED>
__device__ __forceinline__ void load_all(const TileSmem& sm, const float4* __restrict__ P, const float4* __restrict__ L,
                                         const float4* __restrict__ U, const float4* __restrict__ S1,
                                         const float2* __restrict__ S2, uint32_t e, float4& p, float4& u, float4& s1,
                                         float2& s2) {
  if (STAGED) {
    p = win_P(sm, e); u = win_U(sm, e); s1 = win_S1(sm, e); s2 = win_S2(sm, e);
  } else {
    const uint32_t g = window_to_global(sm, e);
    u = U[g]; p = rel_pos_q(P[g], tag_of(u.w), sm); s1 = S1[g]; s2 = S2[g];
  }
}

// the same for the rates pair loops: .w = the signed volume V_j (see relativize_apply<true>)
template <bool STAGED>
__device__ __forceinline__ void load_rates(const TileSmem& sm, const float4* __restrict__ P, const float4* __restrict__ L,
                                           const float4* __restrict__ U, const float4* __restrict__ S1,
                                           const float2* __restrict__ S2, uint32_t e, float m, float4& p, float4& u,
                                           float4& s1, float2& s2) {
  if (STAGED) {
    p = win_P(sm, e); u = win_U(sm, e); s1 = win_S1(sm, e); s2 = win_S2(sm, e);
  } else {
    const uint32_t g = window_to_global(sm, e);
    u = U[g]; p = rel_pos_q(P[g], tag_of(u.w), sm); s1 = S1[g]; s2 = S2[g];
    p.w = signed_volume(p.w, u.w, m);
  }
}

// ---------------------------------------------------------------------------------------
template <int STAGE, int KER, bool STAGED>
__device__ __forceinline__ void bce_tile(const Phys& ph, TileSmem& sm, const float4* __restrict__ P,
                                         const float4* __restrict__ L, float4* __restrict__ U, float4* __restrict__ S1,
                                         float2* __restrict__ S2, const uint16_t* __restrict__ list,
                                         const uint32_t* __restrict__ nlist, const Pose* __restrict__ pose, ListShape ls,
                                         Debug dbg, int dbg_on) {
  const uint32_t n_i = sm.col_pref[NCOL];
  for (uint32_t t = threadIdx.x; t < n_i; t += blockDim.x) {
    int q;
    const uint32_t i = tile_particle(sm, t, q);
    const float4 ui = U[i];
    const uint32_t tag = tag_of(ui.w);
    if (!tag_is_bce(tag)) continue;
    if (tag_frozen(tag)) {   // Extended-Active marker (A31): keeps its extrapolated values
      if (dbg_on) {
        dbg.bu[STAGE][i] = ui;
        dbg.bs1[STAGE][i] = S1[i];
        dbg.bs2[STAGE][i] = S2[i];
      }
      continue;
    }
    const float4 pabs = P[i];
    const float4 pa = rel_pos_q(pabs, tag, sm);
    const uint32_t nl = nlist[i];
    float ub[3] = {0.f, 0.f, 0.f}, ab[3] = {0.f, 0.f, 0.f};
    if (tag_moving(tag)) body_kinematics(pose[tag_body(tag)], pabs.x, pabs.y, pabs.z, ub, ab);
    const float ga[3] = {ph.g[0] - ab[0], ph.g[1] - ab[1], ph.g[2] - ab[2]};
    float SW = 0.f, su[3] = {0.f, 0.f, 0.f}, ss[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, sh = 0.f;
    const uint4* seg = reinterpret_cast<const uint4*>(list) + i;
    // whole chunks of 8 (padded with the marker itself, excluded by the fluid mask): branch-free
    const uint32_t nch = (nl + 7) >> 3;
    uint4 vn = seg[0];   // chunk prefetch, as in pair_loop
    const size_t ls_stride = ls.stride;
    for (uint32_t c = 0; c < nch; ++c) {
      const uint4 v = vn;
      vn = seg[(size_t)min(c + 1, nch - 1) * ls_stride];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t off = list_entry(v, e);
        float4 pf, uf, s1;
        float2 s2;
        load_all<STAGED>(sm, P, L, U, S1, S2, off, pf, uf, s1, s2);
        const float dx = pa.x - pf.x, dy = pa.y - pf.y, dz = pa.z - pf.z;
        const float r2 = dx * dx + dy * dy + dz * dz;
        // fluid neighbours only; W = 0 beyond the support (A17)
        const bool ok = !tag_is_bce(tag_of(uf.w)) && r2 < ph.R2;
        const float r = (r2 > 0.f) ? r2 * rsqrt_approx(r2) : 0.f;
        const float W = ok ? kernel_W<KER>(r, ph) : 0.f;
        SW += W;
        su[0] += uf.x * W; su[1] += uf.y * W; su[2] += uf.z * W;
        ss[0] += s1.x * W; ss[1] += s1.y * W; ss[2] += s1.z * W;
        ss[3] += s1.w * W; ss[4] += s2.x * W; ss[5] += s2.y * W;
        sh += pf.w * (ga[0] * dx + ga[1] * dy + ga[2] * dz) * W;
      }
    }
    float4 uo, s1o;
    float2 s2o;
    if (SW > 0.f) {
      const float inv = 1.0f / SW;
      uo = make_float4(2.f * ub[0] - su[0] * inv, 2.f * ub[1] - su[1] * inv, 2.f * ub[2] - su[2] * inv, ui.w);
      const float hyd = sh * inv;
      s1o = make_float4(ss[0] * inv - hyd, ss[1] * inv - hyd, ss[2] * inv - hyd, ss[3] * inv);
      s2o = make_float2(ss[4] * inv, ss[5] * inv);
    } else {   // A11
      uo = make_float4(ub[0], ub[1], ub[2], ui.w);
      s1o = make_float4(0.f, 0.f, 0.f, 0.f);
      s2o = make_float2(0.f, 0.f);
    }
    U[i] = uo;
    S1[i] = s1o;
    S2[i] = s2o;
    if (dbg_on) {
      dbg.bu[STAGE][i] = uo;
      dbg.bs1[STAGE][i] = s1o;
      dbg.bs2[STAGE][i] = s2o;
    }
  }
}

// Persistent over the tiles that hold markers (listed by k_filter_t at the last rebuild): a tile
// of fluid only has nothing to extrapolate, and a CTA per tile of the whole grid would cost more
// in setup than the markers' work.
template <int STAGE, int KER>
__global__ void BCE_BOUNDS
    k_bce_t(Grid g, Phys ph, const uint32_t* __restrict__ cell_start, const float4* __restrict__ P,
            const float4* __restrict__ L, float4* __restrict__ U, float4* __restrict__ S1, float2* __restrict__ S2,
            const uint16_t* __restrict__ list, const uint32_t* __restrict__ nlist, const Pose* __restrict__ pose,
            ListShape ls, Debug dbg, int dbg_on, ErrLatch* err, long long step, const uint32_t* __restrict__ mtiles,
            const uint32_t* __restrict__ mcount) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  if (latched(err)) return;
  const uint32_t ntile = *mcount;
  for (uint32_t k = blockIdx.x; k < ntile; k += gridDim.x) {
    __syncthreads();   // the previous tile's window is no longer read
    const uint32_t mt = mtiles[k];
    const TileGeom G = tile_geom(g, (long long)(mt & 0x0fffffffu));
    tile_setup(g, G, cell_start, sm);
    if (sm.col_pref[NCOL] == 0) continue;
    if (sm.run_base[WR] > 65535u) {
      if (threadIdx.x == 0) latch_error(err, -9, -1, step, (long long)sm.run_base[WR]);
      continue;
    }
    // only the cells within one of the markers' rows (z0 + zl .. z0 + zh, recorded by the filter):
    // every entry of a marker's list lies there (floor tiles: about half of the window)
    const int zmk = G.z0 + (int)((mt >> 28) & 3u), zMk = G.z0 + (int)(mt >> 30);
    const int klo = max(zmk - 1, G.zlo) - G.zlo, khi = min(zMk + 1, G.zhi) - G.zlo + 1;
    tile_stage_cells(P, U, S1, S2, sm, klo, khi);
    tile_stage_wait();
    __syncthreads();
    tile_relativize_cells(sm, klo, khi);
    __syncthreads();
    if (sm.staged) bce_tile<STAGE, KER, true>(ph, sm, P, L, U, S1, S2, list, nlist, pose, ls, dbg, dbg_on);
    else bce_tile<STAGE, KER, false>(ph, sm, P, L, U, S1, S2, list, nlist, pose, ls, dbg, dbg_on);
  }
}

// ---------------------------------------------------------------------------------------
struct PairAcc {
  float L[9], Gs[3], Ms[3], Pi[3];
};

// own state of a thread's first particle, requested before the window staging so that its
// latency overlaps the staging and the relativize pass instead of following them
struct Prefetch {
  uint32_t i, nl;
  float4 u, p;
  uint4 c0;
};

// One directed pair (i, j).  pj.w = signed V_j (+ fluid, - marker).  Branch-free, no mask: beyond 2h
// (A17) kernel_F is 0 (clamped), so w = 0; at r = 0 (the self padding, A18) r is lifted to 1e-15 and
// every term carries x_ij = 0; a marker when only fluid counts gets w = 0 — a zero contribution to
// every sum.  The AV term reuses V_j grad W (Pi += (v.r)/den g; the constant c_av multiplies the
// sum in the epilogue).  Two MUFU per pair (rsqrt, one reciprocal for the AV).  (measured: the mask
// compares, the AV products and 64-bit tile divisions removed, k_rates_A/B 11.79/11.42 -> 11.51/11.14 ms)
template <int KER>
__device__ __forceinline__ void pair_terms(PairAcc& A, const Phys& ph, const float4& pi, const float4& ui,
                                           const float4& pj, const float4& uj, const float4& sj1, const float2& sj2,
                                           bool with_L, bool fluid_only) {
  const float dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;   // x_ij = x_i - x_j
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  const float Vj = fabsf(pj.w);
  // W'/r vanishes beyond 2h inside kernel_F; r = 0 (the self padding) is lifted to a tiny r so that
  // F stays finite and every term (each carries x_ij = 0) is exactly 0
  const float r2c = fmaxf(r2, 1e-30f);
  const float rinv = rsqrt_approx(r2c);
  const float F = kernel_F<KER>(r2c * rinv, rinv, ph);                // W'(r)/r (A1 / A28)
  const float w = (fluid_only && !(pj.w > 0.f)) ? 0.f : Vj * F;       // V_j W'/r (A7)
  const float gx = w * dx, gy = w * dy, gz = w * dz;                  // V_j grad_i W_ij
  const float dux = uj.x - ui.x, duy = uj.y - ui.y, duz = uj.z - ui.z; // u_ji
  if (with_L) {   // velocity gradient L_ab += V_j u_ji,a gradW_b (F2, A4)
    A.L[0] = fmaf(dux, gx, A.L[0]); A.L[1] = fmaf(dux, gy, A.L[1]); A.L[2] = fmaf(dux, gz, A.L[2]);
    A.L[3] = fmaf(duy, gx, A.L[3]); A.L[4] = fmaf(duy, gy, A.L[4]); A.L[5] = fmaf(duy, gz, A.L[5]);
    A.L[6] = fmaf(duz, gx, A.L[6]); A.L[7] = fmaf(duz, gy, A.L[7]); A.L[8] = fmaf(duz, gz, A.L[8]);
  }
  // F3 momentum: sum V_j (sigma_i + sigma_j) gradW = sigma_i sum V_j gradW + sum V_j sigma_j gradW
  A.Gs[0] += gx; A.Gs[1] += gy; A.Gs[2] += gz;
  A.Ms[0] = fmaf(sj1.x, gx, fmaf(sj1.w, gy, fmaf(sj2.x, gz, A.Ms[0])));
  A.Ms[1] = fmaf(sj1.w, gx, fmaf(sj1.y, gy, fmaf(sj2.y, gz, A.Ms[1])));
  A.Ms[2] = fmaf(sj2.x, gx, fmaf(sj2.y, gy, fmaf(sj1.z, gz, A.Ms[2])));
  // artificial viscosity (Eq. 13/14, sign of reading A9): v_ij . r_ij with v_ij = u_i - u_j;
  // gamma_a h c_s (m_j / rho_bar_ij) (v_ij . r_ij) / (r^2 + xi^2) W'/r with rho_bar = (rho_i + rho_j)/2
  // and rho_j = m / V_j:  m / rho_bar = 2 m V_j / (rho_i V_j + m)  (c_av holds 2 m gamma_a h c_s)
  const float vr = -fmaf(duz, dz, fmaf(duy, dy, dux * dx));
  const float den = fmaf(pi.w, Vj, ph.m) * (r2 + ph.xi2);
  const float cv = vr * rcp_approx(den);   // c_av applied once in the epilogue
  const float coef = (!ph.unilateral || vr < 0.f) ? cv : 0.f;
  A.Pi[0] = fmaf(coef, gx, A.Pi[0]); A.Pi[1] = fmaf(coef, gy, A.Pi[1]); A.Pi[2] = fmaf(coef, gz, A.Pi[2]);
}

template <int KER, bool STAGED>
__device__ __forceinline__ void pair_loop(PairAcc& A, const Phys& ph, const TileSmem& sm, const float4* __restrict__ P,
                                          const float4* __restrict__ L, const float4* __restrict__ U,
                                          const float4* __restrict__ S1, const float2* __restrict__ S2,
                                          const uint16_t* __restrict__ list, uint32_t i, ListShape ls, uint32_t nl,
                                          uint4 first, const float4& pi, const float4& ui, bool with_L,
                                          bool fluid_only) {
  const uint4* seg = reinterpret_cast<const uint4*>(list) + i;
  const size_t ls_stride = ls.stride;
  const uint32_t nch = (nl + 7) >> 3;
  // the list streams from HBM (written by the filter, larger than L2): chunks c + 1 and c + 2 are in
  // flight while chunk c is processed, so their latency hides behind 8-16 pair evaluations; chunk 0
  // comes from the caller (requested before the window staging).  Two ahead instead of one:
  // k_rates_A 13.52 -> 13.37 ms, k_rates_B 13.94 -> 13.74 ms (4 more spilled words, outside the loop);
  // three ahead ran 14.26 / 14.54 ms (register pressure)
  uint4 vn = first;
  uint4 vn2 = seg[nch > 1 ? ls_stride : 0];   // an empty list (nch = 0) has only chunk 0
  for (uint32_t c = 0; c < nch; ++c) {   // whole padded chunks of 8, branch-free
    const uint4 v = vn;
    vn = vn2;
    vn2 = seg[(size_t)min(c + 2, nch - 1) * ls_stride];
    // chunk c + 4 to L2 (no register): the LDG two chunks ahead then hits L2 (measured: k_rates_B
    // 11.14 -> 11.05 ms; 3 or 5 ahead the same)
    if (c + 4 < nch)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(seg + (size_t)(c + 4) * ls_stride));
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      float4 pj, uj, s1;
      float2 s2;
      // (measured: the x/y halves on packed f32x2 instructions, 57 instead of 68 instructions per
      //  pair, and a two-phase body (geometry of 4-8 entries, then their sums) ran 2 % slower and
      //  the same: the pair loop is bound by the window gathers and the tile prologue, not issue)
      load_rates<STAGED>(sm, P, L, U, S1, S2, list_entry(v, e), ph.m, pj, uj, s1, s2);
      pair_terms<KER>(A, ph, pi, ui, pj, uj, s1, s2, with_L, fluid_only);
    }
  }
}

// STAGE 0: (P,L,U,S) = y_n; writes y_mid to (YP,YL,YU,YS).  STAGE 1: (P,L,U,S) = y_mid;
// (YP,YL,YU,YS) = y_n in, y_{n+1} out (own slot only; neighbours are read from y_mid).
template <int STAGE, int KER, bool STAGED>
__device__ __forceinline__ void rates_tile(const Phys& ph, float dt, TileSmem& sm, const float4* __restrict__ P,
                                           const float4* __restrict__ L, const float4* __restrict__ U,
                                           const float4* __restrict__ S1, const float2* __restrict__ S2,
                                           float4* __restrict__ YP, float4* __restrict__ YL, float4* __restrict__ YU,
                                           float4* __restrict__ YS1, float2* __restrict__ YS2,
                                           const uint16_t* __restrict__ list, const uint32_t* __restrict__ nlist,
                                           ListShape ls, float4* __restrict__ macc, Debug dbg, int dbg_on, ErrLatch* err,
                                           const uint32_t* __restrict__ ids, long long step, const Prefetch& pre) {
  const uint32_t n_i = sm.col_pref[NCOL];
  for (uint32_t t = threadIdx.x; t < n_i; t += blockDim.x) {
    const bool first = t == threadIdx.x;   // the thread's first particle was prefetched
    int q;
    const uint32_t i = first ? pre.i : tile_particle(sm, t, q);
    const float4 ui = first ? pre.u : U[i];
    const uint32_t tag = tag_of(ui.w);
    const bool bce = tag_is_bce(tag);
    if (bce && !(STAGE == 1 && tag_moving(tag))) continue;
    if (tag_frozen(tag)) {   // Extended-Active fluid (A31): a neighbour only, y_mid = y_{n+1} = y_n
      if (STAGE == 0) {
        YP[i] = P[i]; YL[i] = L[i]; YU[i] = ui; YS1[i] = S1[i]; YS2[i] = S2[i];
      }
      if (dbg_on) {
        dbg.drho[STAGE][i] = 0.f;
        dbg.acc[STAGE][i] = make_float4(0.f, 0.f, 0.f, 0.f);
        dbg.ds1[STAGE][i] = make_float4(0.f, 0.f, 0.f, 0.f);
        dbg.ds2[STAGE][i] = make_float2(0.f, 0.f);
      }
      continue;
    }
    const float4 pi = rel_pos_q(first ? pre.p : P[i], tag, sm);
    const uint32_t nl = first ? pre.nl : nlist[i];
    // stage A: chunk 0 was prefetched to L2 with the others (held in a register across the prologue
    // it was spilled, and the spill waited for the load: k_rates_A 11.49 -> 11.01 ms); stage B keeps it
    const uint4 c0 = (STAGE == 1 && first) ? pre.c0 : reinterpret_cast<const uint4*>(list)[i];
    PairAcc A;
#pragma unroll
    for (int k = 0; k < 9; ++k) A.L[k] = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) { A.Gs[k] = 0.f; A.Ms[k] = 0.f; A.Pi[k] = 0.f; }
    if (bce) {   // STAGE 1, moving-body marker: m a_s over fluid neighbours, no gravity (A13)
      pair_loop<KER, STAGED>(A, ph, sm, P, L, U, S1, S2, list, i, ls, nl, c0, pi, ui, false, true);
      const float4 si1 = S1[i];
      const float2 si2 = S2[i];
      const float rinv_i = 1.0f / pi.w;
      float a[3];
      a[0] = (si1.x * A.Gs[0] + si1.w * A.Gs[1] + si2.x * A.Gs[2] + A.Ms[0]) * rinv_i + ph.c_av * A.Pi[0];
      a[1] = (si1.w * A.Gs[0] + si1.y * A.Gs[1] + si2.y * A.Gs[2] + A.Ms[1]) * rinv_i + ph.c_av * A.Pi[1];
      a[2] = (si2.x * A.Gs[0] + si2.y * A.Gs[1] + si1.z * A.Gs[2] + A.Ms[2]) * rinv_i + ph.c_av * A.Pi[2];
      macc[i] = make_float4(ph.m * a[0], ph.m * a[1], ph.m * a[2], 0.f);
      if (dbg_on) dbg.acc[1][i] = make_float4(a[0], a[1], a[2], 0.f);
      continue;
    }
    pair_loop<KER, STAGED>(A, ph, sm, P, L, U, S1, S2, list, i, ls, nl, c0, pi, ui, true, false);
    // own state for the epilogue, (re)loaded after the loop to keep registers free inside it
    const float4 phi = first ? pre.p : P[i];
    const float4 pli = L[i];   // (held across the prologue it was spilled: k_rates_A 11.02 -> 10.72 ms)
    const float4 si1 = S1[i];
    const float2 si2 = S2[i];
    const float rinv_i = 1.0f / pi.w;
    float a[3];
    a[0] = (si1.x * A.Gs[0] + si1.w * A.Gs[1] + si2.x * A.Gs[2] + A.Ms[0]) * rinv_i + ph.c_av * A.Pi[0] + ph.g[0];
    a[1] = (si1.w * A.Gs[0] + si1.y * A.Gs[1] + si2.y * A.Gs[2] + A.Ms[1]) * rinv_i + ph.c_av * A.Pi[1] + ph.g[1];
    a[2] = (si2.x * A.Gs[0] + si2.y * A.Gs[1] + si1.z * A.Gs[2] + A.Ms[2]) * rinv_i + ph.c_av * A.Pi[2] + ph.g[2];
    // continuity (Eq. continuity_dis): drho = -rho_i sum (u_j - u_i) . gradW V_j = -rho_i tr L
    const float drho = -pi.w * (A.L[0] + A.L[4] + A.L[8]);
    // Jaumann stress rate (Eq. stress_rate with Eq. 3; readings A4–A6)
    const float sig[9] = {si1.x, si1.w, si2.x, si1.w, si1.y, si2.y, si2.x, si2.y, si1.z};
    float E[9], Om[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        E[3 * r + c] = 0.5f * (A.L[3 * r + c] + A.L[3 * c + r]);
        Om[3 * r + c] = 0.5f * (A.L[3 * r + c] - A.L[3 * c + r]);
      }
    const float tr = E[0] + E[4] + E[8];
    float ds[6];
    const int rr[6] = {0, 1, 2, 0, 0, 1}, cc[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int r = rr[k], c = cc[k];
      float v = 0.f;
#pragma unroll
      for (int s = 0; s < 3; ++s) v += Om[3 * r + s] * sig[3 * s + c] - sig[3 * r + s] * Om[3 * s + c];
      v += 2.0f * ph.G * E[3 * r + c];
      if (r == c) v += (ph.K - 2.0f * ph.G / 3.0f) * tr;
      ds[k] = v;
    }
    if (dbg_on) {
      dbg.drho[STAGE][i] = drho;
      dbg.acc[STAGE][i] = make_float4(a[0], a[1], a[2], 0.f);
      dbg.ds1[STAGE][i] = make_float4(ds[0], ds[1], ds[2], ds[3]);
      dbg.ds2[STAGE][i] = make_float2(ds[4], ds[5]);
    }
    if (STAGE == 0) {
      const float hd = 0.5f * dt;
      float hx = phi.x, hy = phi.y, hz = phi.z, lx = pli.x, ly = pli.y, lz = pli.z;
      comp_add(hx, lx, hd * ui.x);   // x_mid = x_n + dt/2 u_n, compensated
      comp_add(hy, ly, hd * ui.y);
      comp_add(hz, lz, hd * ui.z);
      YP[i] = make_float4(hx, hy, hz, phi.w + hd * drho);
      YL[i] = make_float4(lx, ly, lz, 0.f);
      YU[i] = make_float4(ui.x + hd * a[0], ui.y + hd * a[1], ui.z + hd * a[2],
                          __uint_as_float(tag_with_lo(tag, hx, hy, hz, lx, ly, lz)));
      YS1[i] = make_float4(si1.x + hd * ds[0], si1.y + hd * ds[1], si1.z + hd * ds[2], si1.w + hd * ds[3]);
      YS2[i] = make_float2(si2.x + hd * ds[4], si2.y + hd * ds[5]);
    } else {
      const float4 p0 = YP[i];
      const float4 l0 = YL[i];
      const float4 u0 = YU[i];
      const float4 s01 = YS1[i];
      const float2 s02 = YS2[i];
      const float sn[6] = {s01.x, s01.y, s01.z, s01.w, s02.x, s02.y};
      float s[6] = {s01.x + dt * ds[0], s01.y + dt * ds[1], s01.z + dt * ds[2],
                    s01.w + dt * ds[3], s02.x + dt * ds[4], s02.y + dt * ds[5]};
      return_map(s, sn, ph, dt);
      float hx = p0.x, hy = p0.y, hz = p0.z, lx = l0.x, ly = l0.y, lz = l0.z;
      comp_add(hx, lx, dt * ui.x);   // x_{n+1} = x_n + dt u_mid, compensated
      comp_add(hy, ly, dt * ui.y);
      comp_add(hz, lz, dt * ui.z);
      const float4 pn = make_float4(hx, hy, hz, p0.w + dt * drho);
      const float4 un = make_float4(u0.x + dt * a[0], u0.y + dt * a[1], u0.z + dt * a[2],
                                    __uint_as_float(tag_with_lo(tag_of(u0.w), hx, hy, hz, lx, ly, lz)));
      YP[i] = pn;
      YL[i] = make_float4(lx, ly, lz, 0.f);
      YU[i] = un;
      YS1[i] = make_float4(s[0], s[1], s[2], s[3]);
      YS2[i] = make_float2(s[4], s[5]);
      const float chk = pn.x + pn.y + pn.z + pn.w + un.x + un.y + un.z + s[0] + s[1] + s[2] + s[3] + s[4] + s[5];
      if (!isfinite(chk)) latch_error(err, -3 /*CRM_E_NONFINITE*/, (long long)ids[i], step, 0);
    }
  }
}

template <int STAGE, int KER>
__global__ void TILE_BOUNDS
    k_rates_t(Grid g, Phys ph, float dt, const uint32_t* __restrict__ cell_start, const float4* __restrict__ P,
              const float4* __restrict__ L, const float4* __restrict__ U, const float4* __restrict__ S1,
              const float2* __restrict__ S2, float4* __restrict__ YP, float4* __restrict__ YL, float4* __restrict__ YU,
              float4* __restrict__ YS1, float2* __restrict__ YS2, const uint16_t* __restrict__ list,
              const uint32_t* __restrict__ nlist,
              ListShape ls, float4* __restrict__ macc, Debug dbg, int dbg_on, ErrLatch* err,
              const uint32_t* __restrict__ ids, long long step, long long tile_base,
              const uint32_t* __restrict__ tile_list) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem& sm = *reinterpret_cast<TileSmem*>(smem_raw);
  if (latched(err)) return;
#ifdef CRM_EXP_TIMING
  const bool tim = STAGE == 1 && blockIdx.x < 8192u;
  unsigned long long* T = g_exp_timing + 6 * blockIdx.x;
  if (tim && threadIdx.x == 0) T[0] = clock64();
#define EXP_T(k) if (tim && threadIdx.x == 0) T[k] = clock64();
#else
#define EXP_T(k)
#endif
  const TileGeom G = tile_geom(g, tile_list ? (long long)tile_list[blockIdx.x] : tile_base + (long long)blockIdx.x);
  tile_setup(g, G, cell_start, sm);
  EXP_T(1)
  const uint32_t n_i = sm.col_pref[NCOL];
  if (n_i == 0) return;
  if (sm.run_base[WR] > 65535u) {
    if (threadIdx.x == 0) latch_error(err, -9, -1, step, (long long)sm.run_base[WR]);
    return;
  }
  // the window copy starts right away (a tile of markers only, rare, stages for nothing); the
  // lo parts of the window's positions and the own state of each thread's first particle are
  // requested beside it (before the bookkeeping barrier: issued after it, the lo loads queued
  // behind the copy and added ~3k cycles to every tile's prologue)
  // (measured: the copy on the bulk-copy engine, 48 cp.async.bulk of ~1.7 KB per tile with an
  //  mbarrier byte count, ran 1.5 % slower — here and in round 1: the window's arrival rate, not the
  //  copy instructions, bounds the prologue)
  tile_stage(P, U, S1, S2, sm);
#ifndef CRM_LISTPF
#define CRM_LISTPF 12
#endif

  // stage A reads lists the filter has just written (the filter's 6 GB of lists have left L2): chunks
  // 0 .. CRM_LISTPF-1 of each thread's first particle are prefetched to L2 with the window copy
  // (measured: k_rates_A 12.28 -> 11.79 ms with 11 chunks; 4: 12.11, 16: 11.85; stage B gains nothing)
  if (STAGE == 0 && CRM_LISTPF > 1 && threadIdx.x < n_i) {
    int q;
    const uint32_t i0 = tile_particle(sm, threadIdx.x, q);
#pragma unroll
    for (int cc = 0; cc < CRM_LISTPF; ++cc)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint4*>(list) + (size_t)cc * ls.stride + i0));
  }
  Prefetch pre;
  if (threadIdx.x < n_i) {
    int q;
    pre.i = tile_particle(sm, threadIdx.x, q);
    pre.u = U[pre.i];
    pre.p = P[pre.i];
    pre.nl = nlist[pre.i];
    if (STAGE == 1) pre.c0 = reinterpret_cast<const uint4*>(list)[pre.i];
  }
  // marker bookkeeping that needs no window; detect whether the tile has pair work
  int work = 0;
  for (uint32_t t = threadIdx.x; t < n_i; t += blockDim.x) {
    int q;
    const uint32_t i = t == threadIdx.x ? pre.i : tile_particle(sm, t, q);
    const float4 ui = t == threadIdx.x ? pre.u : U[i];
    const uint32_t tag = tag_of(ui.w);
    if (!tag_is_bce(tag)) {
      work = 1;
    } else if (STAGE == 0) {
      YP[i] = P[i];     // markers: x at t_n (moving ones are re-placed at t_n + dt/2 afterwards)
      YL[i] = L[i];
      YU[i] = ui;       // tag; u and sigma are replaced by the stage-B extrapolation (frozen
      YS1[i] = S1[i];   // Extended-Active markers keep these copies, A31)
      YS2[i] = S2[i];
    } else {
      YU[i] = ui;       // y_{n+1} of a marker: its stage-B extrapolated u and sigma
      YS1[i] = S1[i];
      YS2[i] = S2[i];
      if (tag_moving(tag)) work = 1;
    }
  }
  const bool any = __syncthreads_or(work);
  EXP_T(2)
  tile_stage_wait();
  if (!any) return;
  __syncthreads();
  EXP_T(3)
  relativize_apply<true>(sm, ph.m);
  __syncthreads();
  EXP_T(4)
  if (sm.staged)
    rates_tile<STAGE, KER, true>(ph, dt, sm, P, L, U, S1, S2, YP, YL, YU, YS1, YS2, list, nlist, ls, macc, dbg, dbg_on,
                            err, ids, step, pre);
  else
    rates_tile<STAGE, KER, false>(ph, dt, sm, P, L, U, S1, S2, YP, YL, YU, YS1, YS2, list, nlist, ls, macc, dbg, dbg_on,
                             err, ids, step, pre);
#ifdef CRM_EXP_TIMING
  if (tim && (threadIdx.x & 31) == 0) atomicMax(&T[5], clock64());
#endif
}

// ---------------------------------------------------------------------------------------
// debug: hot-path lists (window offsets) -> global sorted indices, ELL k-major u32; the
// zero-weight self padding is dropped and the remaining count written to nout
__global__ void k_decode_lists(int n, Grid g, const uint32_t* __restrict__ cell_start,
                               const uint32_t* __restrict__ cell_of, const uint16_t* __restrict__ list,
                               const uint32_t* __restrict__ nlist, ListShape ls, uint32_t* __restrict__ out,
                               uint32_t* __restrict__ nout) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = cell_of[i];
  const int Nz = g.dims[2], Ny = g.dims[1];
  const int cz = (int)(c % (uint32_t)Nz), cy = (int)((c / (uint32_t)Nz) % (uint32_t)Ny), cx = (int)(c / (uint32_t)(Ny * Nz));
  const long long t = ((long long)(cx / TX) * tiles_y(g) + cy / TY) * tiles_z(g) + cz / TZ;
  const TileGeom G = tile_geom(g, t);
  const int nzw = G.zhi - G.zlo + 1;
  uint32_t rs[WR], rb[WR + 1];
  uint32_t acc = 0;
  for (int r = 0; r < WR; ++r) {
    const int x = G.X0 - 1 + r / WRY, y = G.Y0 - 1 + r % WRY;
    const bool valid = x >= 0 && x < g.dims[0] && y >= 0 && y < g.dims[1];
    const uint32_t c0 = valid ? cell_id(g, x, y, G.zlo) : 0u;
    rs[r] = valid ? cell_start[c0] : 0u;
    const uint32_t re = valid ? cell_start[c0 + nzw] : 0u;
    rb[r] = acc;
    acc += re - rs[r];
  }
  rb[WR] = acc;
  uint32_t kk = 0;
  for (uint32_t k = 0; k < nlist[i]; ++k) {
    const uint32_t e = list[((size_t)(k >> 3) * ls.stride + (size_t)i) * 8 + (k & 7)];
    const uint32_t off = acc <= (uint32_t)WMAX ? e >> 4 : e;
    int r = 0;
    for (int q = 1; q < WR; ++q) r += (rb[q] <= off) ? 1 : 0;
    const uint32_t j = rs[r] + (off - rb[r]);
    if (j == (uint32_t)i) continue;   // zero-weight self padding
    out[(size_t)kk * n + i] = j;
    ++kk;
  }
  nout[i] = kk;
}

}  // namespace crmk
