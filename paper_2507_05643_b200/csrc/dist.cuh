// dist.cuh — multi-GPU slab decomposition along x.
//
// Each rank owns the cell planes [x_lo, x_hi) (boundaries from a prefix sum of per-plane particle
// counts, aligned to the tile width) and keeps one ghost plane (one 2h cell) on each interior
// face.  With the B3 cell order a plane is one contiguous index range of the sorted state, so
// every exchange is a handful of contiguous slices.  Per step:
//   P0  one pass over the local particles (k_slab_pack): last step's ghosts dropped; owned particles
//       now in a neighbour's first plane packed as emigrants (kept here as ghosts); owned particles of
//       the first / last plane packed as the neighbours' ghost planes;      E0  counts
//   P1  E1  payloads (id + 72-B state), appended: immigrants, then ghosts
//   P2  immigrants checked to sit in the boundary plane, received ghosts flagged
//   P4  the one sort of the step (ghosts in, emigrants and old ghosts out), BCE at y_n on owned tiles
//   E4  boundary planes (markers now extrapolated) -> ghosts
//   P5  rates + half step, boundary tile columns     E5  y_mid boundary planes -> ghosts
//   P6  rates + half step, interior columns (overlaps E5 on the NCCL transport)
//   P7  BCE extrapolation at y_mid                   E7  y_mid boundary planes -> ghosts
//   P8  rates + full step + return map on owned tiles
// (Alg. 2 reuse steps skip P0-P2 and the sort and refresh the ghost values in P3.)
// Neighbour iteration order is the global (cell, id) order restricted to the local planes, so
// owned particles follow bit-identical trajectories to a one-GPU run.
// Transports: NCCL point-to-point (ncclSend/ncclRecv in a group, on the context stream; NCCL is
// loaded at run time) or an in-process loopback between contexts of one process (crm_group_step;
// used to test the decomposition on one GPU).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include "context.cuh"

namespace {

// ---------------------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* cands[] = {getenv("CRM_NCCL_LIB"), "libnccl.so.2",
#ifdef CRM_NCCL_DEFAULT
                         CRM_NCCL_DEFAULT,
#endif
                         nullptr};
  void* h = nullptr;
  for (const char* p : cands)
    if (p && (h = dlopen(p, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return api;
#define LD(field, sym) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #sym))
  LD(getUniqueId, ncclGetUniqueId); LD(commInitRank, ncclCommInitRank); LD(commDestroy, ncclCommDestroy);
  LD(send, ncclSend); LD(recv, ncclRecv); LD(groupStart, ncclGroupStart); LD(groupEnd, ncclGroupEnd);
  LD(errorString, ncclGetErrorString);
#undef LD
  api.ok = api.getUniqueId && api.commInitRank && api.send && api.recv && api.groupStart && api.groupEnd;
  return api;
}

// ---------------------------------------------------------------------------------------
void post(crm_t* c, int peer, bool send, const void* ptr, size_t bytes) {
  if (bytes == 0 || peer < 0 || peer >= c->world) return;
  c->posts.push_back({peer, send, const_cast<void*>(ptr), bytes});
}

// state slice [b, e) of buffer set `y` (ids included when with_ids)
void post_slice(crm_t* c, int peer, bool send, int y, uint32_t b, uint32_t e, bool with_ids) {
  if (e <= b) return;
  const size_t k = e - b;
  post(c, peer, send, c->P[y] + b, k * 16);
  post(c, peer, send, c->L[y] + b, k * 16);
  post(c, peer, send, c->U[y] + b, k * 16);
  post(c, peer, send, c->S1[y] + b, k * 16);
  post(c, peer, send, c->S2[y] + b, k * 8);
  if (with_ids) post(c, peer, send, c->ids[y] + b, k * 4);
}

void post_mid_slice(crm_t* c, int peer, bool send, uint32_t b, uint32_t e) {
  if (e <= b) return;
  const size_t k = e - b;
  post(c, peer, send, c->Pm + b, k * 16);
  post(c, peer, send, c->Lm + b, k * 16);
  post(c, peer, send, c->Um + b, k * 16);
  post(c, peer, send, c->S1m + b, k * 16);
  post(c, peer, send, c->S2m + b, k * 8);
}

// the compute stream waits for an asynchronous halo (phase 5's) before touching ghost slots
void wait_comm(crm_t* c) {
  if (!c->comm_pending) return;
  cudaStreamWaitEvent(c->stream, c->ev_comm, 0);
  c->comm_pending = false;
}

// NCCL transport: issue every pending transfer of this rank as one group on the stream (or, for the
// y_mid halo of phase 5, on the communication stream after the boundary tiles: it overlaps the
// interior tiles of phase 6)
int nccl_flush(crm_t* c) {
  const bool async = c->halo_async;
  c->halo_async = false;
  if (c->posts.empty()) return CRM_OK;
  NcclApi& api = nccl();
  ncclComm_t comm = (ncclComm_t)c->nccl_comm;
  cudaStream_t st = c->stream;
  if (async) {
    cudaEventRecord(c->ev_boundary, c->stream);
    cudaStreamWaitEvent(c->comm_stream, c->ev_boundary, 0);
    st = c->comm_stream;
  }
  ncclResult_t r = api.groupStart();
  for (const Post& p : c->posts) {
    if (r != ncclSuccess) break;
    r = p.send ? api.send(p.ptr, p.bytes, ncclUint8, p.peer, comm, st)
               : api.recv(p.ptr, p.bytes, ncclUint8, p.peer, comm, st);
  }
  ncclResult_t r2 = api.groupEnd();
  c->posts.clear();
  if (async) {
    cudaEventRecord(c->ev_comm, c->comm_stream);
    c->comm_pending = true;
  }
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(c, CRM_E_COMM, std::string("NCCL: ") + (api.errorString ? api.errorString(r != ncclSuccess ? r : r2) : "error"));
  return CRM_OK;
}

// loopback transport: match every send of rank a to rank b with b's receives from a (FIFO)
int loopback_flush(crm_t** cs, int world) {
  for (int a = 0; a < world; ++a) cs[a]->halo_async = false;   // one shared stream: serial copies
  std::vector<std::vector<size_t>> used(world);
  for (int a = 0; a < world; ++a) used[a].assign(cs[a]->posts.size(), 0);
  for (int a = 0; a < world; ++a) {
    crm_t* c = cs[a];
    for (const Post& s : c->posts) {
      if (!s.send) continue;
      crm_t* d = cs[s.peer];
      bool found = false;
      for (size_t k = 0; k < d->posts.size(); ++k) {
        const Post& r = d->posts[k];
        if (r.send || r.peer != a || used[s.peer][k]) continue;
        if (r.bytes != s.bytes)
          return fail(c, CRM_E_COMM, "loopback: size mismatch " + std::to_string(s.bytes) + " vs " + std::to_string(r.bytes));
        used[s.peer][k] = 1;
        CK(cudaMemcpyAsync(r.ptr, s.ptr, s.bytes, cudaMemcpyDeviceToDevice, c->stream));
        found = true;
        break;
      }
      if (!found) return fail(c, CRM_E_COMM, "loopback: unmatched send");
    }
  }
  for (int a = 0; a < world; ++a) {
    for (size_t k = 0; k < cs[a]->posts.size(); ++k)
      if (!cs[a]->posts[k].send && !used[a][k]) return fail(cs[a], CRM_E_COMM, "loopback: unmatched receive");
    cs[a]->posts.clear();
  }
  return CRM_OK;
}

// ---------------------------------------------------------------------------------------
// slab partition: boundaries at multiples of `align` with ~equal particle counts
int slab_partition(const int64_t* counts, int nplanes, int world, int align, int* bounds) {
  if (world < 1 || align < 1 || nplanes < world * align) return CRM_E_INVALID;
  std::vector<int64_t> cum(nplanes + 1, 0);
  for (int p = 0; p < nplanes; ++p) cum[p + 1] = cum[p] + counts[p];
  const int64_t total = cum[nplanes];
  bounds[0] = 0;
  for (int k = 1; k < world; ++k) {
    const int64_t target = (total * k + world / 2) / world;
    const int lo = bounds[k - 1] + align;
    const int hi = ((nplanes - (world - k) * align) / align) * align;
    int b = lo;
    while (b + align <= hi && cum[b] < target) b += align;
    // take the closer of b and b - align
    if (b - align >= lo && target - cum[b - align] < cum[b] - target) b -= align;
    bounds[k] = std::min(std::max(b, lo), hi);
  }
  bounds[world] = nplanes;
  return CRM_OK;
}

uint32_t plane_start_index(const crm_t* c, int p) {   // cell index of the first cell of plane p
  const long long NyNz = (long long)c->grid.dims[1] * c->grid.dims[2];
  if (p <= 0) return 0;
  if (p >= c->grid.dims[0]) return c->grid.M;
  return (uint32_t)(p * NyNz);
}

// read cellStart at the first cell of planes ps[0..k) (k <= 8) into out
int read_plane_starts(crm_t* c, const int* ps, int k, uint32_t* out) {
  for (int j = 0; j < k; ++j)
    CK(cudaMemcpyAsync(c->h_pin + j, c->cell_start + plane_start_index(c, ps[j]), 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int j = 0; j < k; ++j) out[j] = c->h_pin[j];
  return CRM_OK;
}

// count exchange: two words per direction (d_xcount: send L[2], send R[2], recv L[2], recv R[2])
int read_counts(crm_t* c, uint32_t* l0, uint32_t* l1, uint32_t* r0, uint32_t* r1) {
  CK(cudaMemcpyAsync(c->h_pin + 16, c->d_xcount + 4, 16, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const bool hl = c->rank > 0, hr = c->rank < c->world - 1;
  *l0 = hl ? c->h_pin[16] : 0;
  if (l1) *l1 = hl ? c->h_pin[17] : 0;
  *r0 = hr ? c->h_pin[18] : 0;
  if (r1) *r1 = hr ? c->h_pin[19] : 0;
  return CRM_OK;
}

int post_counts(crm_t* c, uint32_t l0, uint32_t l1, uint32_t r0, uint32_t r1) {
  c->h_pin[24] = l0; c->h_pin[25] = l1; c->h_pin[26] = r0; c->h_pin[27] = r1;
  CK(cudaMemcpyAsync(c->d_xcount, c->h_pin + 24, 16, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->d_xcount + 4, 0, 16, c->stream));
  post(c, c->rank - 1, true, c->d_xcount + 0, 8);
  post(c, c->rank + 1, true, c->d_xcount + 2, 8);
  post(c, c->rank - 1, false, c->d_xcount + 4, 8);
  post(c, c->rank + 1, false, c->d_xcount + 6, 8);
  return CRM_OK;
}

void issue_sort(crm_t* c, long long step, uint32_t drop_mask);
void issue_bce(crm_t* c, int stage, float dt, long long step, int store_all);
void issue_rates(crm_t* c, int stage, float dt, long long step);
void issue_rates_range(crm_t* c, int stage, float dt, long long step, long long first, long long count);
void issue_body_partial(crm_t* c);
void issue_body_finish(crm_t* c);

// ---------------------------------------------------------------------------------------
// the phases of one slab step (each ends with posts; the transport flushes between phases)
int slab_phase(crm_t* c, int k, float dt, long long step) {
  const int L = c->rank - 1, R = c->rank + 1;
  switch (k) {
    case 0: {   // rebuild: one pass packs emigrants and boundary planes per side (no sort here)
      // Alg. 2: between rebuilds the slots, ghost sets and lists stay; only values move (phase 3)
      c->slab_rebuild = !c->lists_valid || (step % c->ps_freq) == 0;
      launch(c, KID_STEP, k_step_begin, dim3(1), dim3(1), c->d_err, step);
      if (!c->slab_rebuild) return CRM_OK;
      const int y = c->cur;
      CK(cudaMemsetAsync(c->pk.cnt, 0, 16, c->stream));
      if (c->nl)
        launch(c, KID_SLAB, k_slab_pack, dim3(blocks(c->nl, 256)), dim3(256), (int)c->nl, (const float4*)c->P[y],
               (const float4*)c->L[y], c->U[y], (const float4*)c->S1[y], (const float2*)c->S2[y],
               (const uint32_t*)c->ids[y], c->grid, c->x_lo, c->x_hi, c->rank > 0 ? 1 : 0,
               c->rank < c->world - 1 ? 1 : 0, c->pk, c->d_err, step);
      CK(cudaMemcpyAsync(c->h_pin + 32, c->pk.cnt, 16, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      for (int k = 0; k < 4; ++k) c->pk_n[k] = c->h_pin[32 + k];
      if (c->pk_n[0] > c->pk.cap_e || c->pk_n[2] > c->pk.cap_e || c->pk_n[1] > c->pk.cap_g || c->pk_n[3] > c->pk.cap_g)
        return fail(c, CRM_E_CAPACITY, "slab pack buffers exceeded (emigrants or boundary plane)");
      return post_counts(c, c->pk_n[0], c->pk_n[1], c->pk_n[2], c->pk_n[3]);
    }
    case 1: {   // rebuild: payloads — emigrants (owned there) and boundary planes (ghosts there), appended
      if (!c->slab_rebuild) return CRM_OK;
      uint32_t el, gl, er, gr;
      if (int r = read_counts(c, &el, &gl, &er, &gr)) return r;
      c->rv_n[0] = el; c->rv_n[1] = gl; c->rv_n[2] = er; c->rv_n[3] = gr;
      const uint32_t nl = (uint32_t)c->nl;
      if ((int64_t)nl + el + gl + er + gr > c->ncap) return fail(c, CRM_E_CAPACITY, "slab capacity exceeded (immigrants + ghosts)");
      const int y = c->cur;
      for (int d = 0; d < 2; ++d) {   // sends: E then G of each side (the receiver posts in the same order)
        const int peer = d == 0 ? L : R;
        const uint32_t ne = c->pk_n[2 * d], ng = c->pk_n[2 * d + 1], g0 = c->pk.cap_e;
        post(c, peer, true, c->pk.P[d], ne * 16); post(c, peer, true, c->pk.L[d], ne * 16);
        post(c, peer, true, c->pk.U[d], ne * 16); post(c, peer, true, c->pk.S1[d], ne * 16);
        post(c, peer, true, c->pk.S2[d], ne * 8); post(c, peer, true, c->pk.id[d], ne * 4);
        post(c, peer, true, c->pk.P[d] + g0, ng * 16); post(c, peer, true, c->pk.L[d] + g0, ng * 16);
        post(c, peer, true, c->pk.U[d] + g0, ng * 16); post(c, peer, true, c->pk.S1[d] + g0, ng * 16);
        post(c, peer, true, c->pk.S2[d] + g0, ng * 8); post(c, peer, true, c->pk.id[d] + g0, ng * 4);
      }
      // receives, appended behind the local particles: [E left][G left][E right][G right]
      const uint32_t a0 = nl, a1 = a0 + el, a2 = a1 + gl, a3 = a2 + er, a4 = a3 + gr;
      post_slice(c, L, false, y, a0, a1, true);
      post_slice(c, L, false, y, a1, a2, true);
      post_slice(c, R, false, y, a2, a3, true);
      post_slice(c, R, false, y, a3, a4, true);
      return CRM_OK;
    }
    case 2: {   // rebuild: immigrants checked to sit in the boundary plane; ghosts flagged
      if (!c->slab_rebuild) return CRM_OK;
      const int y = c->cur;
      const uint32_t nl = (uint32_t)c->nl;
      const uint32_t a0 = nl, a1 = a0 + c->rv_n[0], a2 = a1 + c->rv_n[1], a3 = a2 + c->rv_n[2], a4 = a3 + c->rv_n[3];
      if (a1 > a0)
        launch(c, KID_SLAB, k_check_plane, dim3(blocks(a1 - a0, 256)), dim3(256), (const float4*)c->P[y],
               (const uint32_t*)c->ids[y], a0, a1, c->grid, c->x_lo, c->d_err, step);
      if (a3 > a2)
        launch(c, KID_SLAB, k_check_plane, dim3(blocks(a3 - a2, 256)), dim3(256), (const float4*)c->P[y],
               (const uint32_t*)c->ids[y], a2, a3, c->grid, c->x_hi - 1, c->d_err, step);
      if (a2 > a1) launch(c, KID_SLAB, k_or_tag, dim3(blocks(a2 - a1, 256)), dim3(256), c->U[y], a1, a2, TAG_GHOST);
      if (a4 > a3) launch(c, KID_SLAB, k_or_tag, dim3(blocks(a4 - a3, 256)), dim3(256), c->U[y], a3, a4, TAG_GHOST);
      c->nl = a4;
      return CRM_OK;
    }
    case 3: {   // Alg. 2 reuse step: refresh the ghost values y_n in place
      if (c->slab_rebuild) return CRM_OK;
      const int y = c->cur;
      post_slice(c, L, true, y, c->s_lo, c->s_lo1, false);
      post_slice(c, R, true, y, c->s_hi1, c->s_hi, false);
      post_slice(c, L, false, y, c->s_lom1, c->s_lo, false);
      post_slice(c, R, false, y, c->s_hi, c->s_hip1, false);
      return CRM_OK;
    }
    case 4: {   // ghosts flagged, local sort, BCE at y_n; boundary planes -> ghosts
      if (c->slab_rebuild) {   // the one sort of the rebuild: old ghosts out, emigrants kept as ghosts
        issue_sort(c, step, TAG_DROP);
        const int ps[7] = {c->x_lo - 1, c->x_lo, c->x_lo + 1, c->x_hi - 1, c->x_hi, c->x_hi + 1, c->grid.dims[0]};
        uint32_t st[7];
        if (int r = read_plane_starts(c, ps, 7, st)) return r;
        c->nl = st[6];
        c->s_lom1 = c->rank > 0 ? st[0] : st[1];
        c->s_lo = st[1]; c->s_lo1 = st[2]; c->s_hi1 = st[3]; c->s_hi = st[4];
        c->s_hip1 = c->rank < c->world - 1 ? st[5] : st[4];
        c->n_owned = c->s_hi - c->s_lo;
      } else {   // the refreshed ghost values carried the owners' tags
        const int y0 = c->cur;
        if (c->s_lo > c->s_lom1)
          launch(c, KID_SLAB, k_or_tag, dim3(blocks(c->s_lo - c->s_lom1, 256)), dim3(256), c->U[y0], c->s_lom1, c->s_lo, TAG_GHOST);
        if (c->s_hip1 > c->s_hi)
          launch(c, KID_SLAB, k_or_tag, dim3(blocks(c->s_hip1 - c->s_hi, 256)), dim3(256), c->U[y0], c->s_hi, c->s_hip1, TAG_GHOST);
      }
      c->ph.build_lists = c->slab_rebuild ? 1 : 0;
      c->lists_valid = true;
      issue_bce(c, 0, dt, step, 0);
      const int y = c->cur;
      post_slice(c, L, true, y, c->s_lo, c->s_lo1, false);
      post_slice(c, R, true, y, c->s_hi1, c->s_hi, false);
      post_slice(c, L, false, y, c->s_lom1, c->s_lo, false);
      post_slice(c, R, false, y, c->s_hi, c->s_hip1, false);
      return CRM_OK;
    }
    case 5:   // rates + half step on the boundary tile columns (all tiles with moving bodies); y_mid halo
    case 6:   // rates + half step on the interior tile columns, overlapping the y_mid halo (NCCL)
    case 7: { // BCE at y_mid; y_mid boundary planes -> ghosts
      // Overlap: the ghost planes a neighbour needs are the y_mid of this slab's first and last
      // planes, which lie in its first and last tile columns (TX planes each).  Stage A runs on
      // those columns first, their y_mid goes out on the communication stream while the interior
      // columns compute (the interior reads y_n only and writes owned slots only; the ghost slots
      // the halo fills are read by stage B).  Moving bodies re-place their markers in y_mid after
      // the whole stage A, so that case keeps one launch and a serial halo.
      const long long per_x = (long long)tiles_y(c->grid) * tiles_z(c->grid);
      const long long ntx = per_x ? c->ntiles / per_x : 0;
      const bool split = c->n_moving_markers == 0 && c->boxes.empty() && ntx > 2;
      if (k == 5) {
        // the copies of E4 carried the owners' tags: mark the ghost planes as ghosts again
        const int y = c->cur;
        if (c->s_lo > c->s_lom1)
          launch(c, KID_SLAB, k_or_tag, dim3(blocks(c->s_lo - c->s_lom1, 256)), dim3(256), c->U[y], c->s_lom1, c->s_lo, TAG_GHOST);
        if (c->s_hip1 > c->s_hi)
          launch(c, KID_SLAB, k_or_tag, dim3(blocks(c->s_hip1 - c->s_hi, 256)), dim3(256), c->U[y], c->s_hi, c->s_hip1, TAG_GHOST);
        if (split) {
          issue_rates_range(c, 0, dt, step, 0, per_x);                    // first tile column
          issue_rates_range(c, 0, dt, step, (ntx - 1) * per_x, per_x);    // last tile column
          c->halo_async = true;   // the flush after this phase runs on the communication stream
        } else {
          issue_rates(c, 0, dt, step);
          if (c->n_moving_markers)   // moving markers at the mid-step pose, before the y_mid halo
            launch(c, KID_MARKERS, k_markers_place, dim3(blocks(c->n_moving_markers, 128)), dim3(128),
                   c->n_moving_markers, (const uint32_t*)c->d_moving_ids, (const float4*)c->d_xlocal,
                   (const uint32_t*)c->slot_of_id, (const Pose*)c->d_posem, c->Pm, c->Lm, c->Um);
        }
      } else if (k == 6) {
        if (split) issue_rates_range(c, 0, dt, step, per_x, (ntx - 2) * per_x);
        return CRM_OK;
      } else {
        wait_comm(c);
        issue_bce(c, 1, dt, step, 0);
      }
      post_mid_slice(c, L, true, c->s_lo, c->s_lo1);
      post_mid_slice(c, R, true, c->s_hi1, c->s_hi);
      post_mid_slice(c, L, false, c->s_lom1, c->s_lo);
      post_mid_slice(c, R, false, c->s_hi, c->s_hip1);
      return CRM_OK;
    }
    case 8:   // rates + full step; moving bodies: this slab's partial loads to every other slab
      wait_comm(c);
      issue_rates(c, 1, dt, step);
      if (c->n_moving_bodies) {
        issue_body_partial(c);
        const size_t blk = (size_t)c->n_moving_bodies * 6;
        for (int p = 0; p < c->world; ++p) {
          if (p == c->rank) continue;
          post(c, p, true, c->d_bpart + (size_t)c->rank * blk, blk * sizeof(double));
          post(c, p, false, c->d_bpart + (size_t)p * blk, blk * sizeof(double));
        }
      }
      return CRM_OK;
    case 9:   // moving bodies: loads summed over slabs in rank order (identical on every rank), update
      if (c->n_moving_bodies) issue_body_finish(c);
      return CRM_OK;
  }
  return CRM_OK;
}
constexpr int kSlabPhases = 10;

}  // namespace
