// dist.cuh — multi-GPU slab decomposition along x.
//
// Each rank owns the cell planes [x_lo, x_hi) (boundaries from a prefix sum of per-plane particle
// counts, aligned to the tile width) and keeps one ghost plane (one 2h cell) on each interior
// face.  With the B3 cell order a plane is one contiguous index range of the sorted state.  No
// phase reads the device on the host: the local count lives in d_slab[0], plane ranges are read
// from cellStart inside the kernels, and every transfer has a fixed size.  Per step:
//   P0  one pass over the local particles (k_slab_pack): last step's ghosts dropped; owned particles
//       now in a neighbour's first plane packed as emigrants (kept here as ghosts); owned particles of
//       the first / last plane packed as the neighbours' ghost planes;
//       E0  the counts and the whole pack buffers (fixed capacity) to both neighbours
//   P1  received immigrants and ghosts appended by count (k_slab_counts, k_slab_append: immigrants
//       checked to sit in the boundary plane, ghosts flagged)
//   P4  the one sort of the step (ghosts in, emigrants and old ghosts out), BCE at y_n on owned tiles
//   E4  boundary planes (markers now extrapolated) packed and sent (k_halo_pack), unpacked into the
//       ghost planes at the start of P5 (k_halo_unpack)
//   P5  rates + half step, boundary tile columns     E5  y_mid boundary planes -> ghosts
//   P6  rates + half step, interior columns (overlaps E5 on the NCCL transport)
//   P7  BCE extrapolation at y_mid                   E7  y_mid boundary planes -> ghosts
//   P8  rates + full step + return map on owned tiles
// (Alg. 2 reuse steps skip P0-P1 and the sort and refresh the ghost values of y_n in P3/P4.)  The
// launch sequence is fixed per (buffer parity, rebuild), so the step is captured once as a CUDA
// graph and replayed (crm.cu run_slab_step, group_slab_step).
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

// the whole of side d of a pack / receive buffer set (fixed capacity: entries [0, count))
void post_buf(crm_t* c, int peer, bool send, const SlabPack& b, int d, size_t count, bool with_ids) {
  post(c, peer, send, b.P[d], count * 16);
  post(c, peer, send, b.L[d], count * 16);
  post(c, peer, send, b.U[d], count * 16);
  post(c, peer, send, b.S1[d], count * 16);
  post(c, peer, send, b.S2[d], count * 8);
  if (with_ids) post(c, peer, send, b.id[d], count * 4);
}

// cell ranges of the slab's two boundary planes (ghost = false: the owned first / last plane, sent)
// or of its two ghost planes (ghost = true: received)
HaloSide halo_side(const crm_t* c, bool ghost) {
  HaloSide hs{};
  const int pl[2] = {ghost ? c->x_lo - 1 : c->x_lo, ghost ? c->x_hi : c->x_hi - 1};
  for (int d = 0; d < 2; ++d) {
    hs.on[d] = d == 0 ? (c->rank > 0) : (c->rank < c->world - 1);
    hs.c0[d] = hs.on[d] ? plane_start_index(c, pl[d]) : 0u;
    hs.c1[d] = hs.on[d] ? plane_start_index(c, pl[d] + 1) : 0u;
  }
  return hs;
}

// halo, sender side: the boundary planes of (P, L, U, S1, S2) packed and posted, each side's count
// beside it (d_xcount[0..1] out, [2..3] in); halo_unpack (after the flush) fills the ghost planes
void halo_pack(crm_t* c, const float4* P, const float4* L, const float4* U, const float4* S1, const float2* S2,
               long long step) {
  launch(c, KID_SLAB, k_halo_pack, dim3(2 * c->num_sms, 2), dim3(256), (const uint32_t*)c->cell_start,
         halo_side(c, false), P, L, U, S1, S2, c->pk, c->d_xcount, c->d_err, step);
  for (int d = 0; d < 2; ++d) {
    const int peer = d == 0 ? c->rank - 1 : c->rank + 1;
    post_buf(c, peer, true, c->pk, d, c->pk.cap_g, false);
    post(c, peer, true, c->d_xcount + d, 4);
    post_buf(c, peer, false, c->rv, d, c->rv.cap_g, false);
    post(c, peer, false, c->d_xcount + 2 + d, 4);
  }
}
void halo_unpack(crm_t* c, float4* P, float4* L, float4* U, float4* S1, float2* S2, long long step) {
  launch(c, KID_SLAB, k_halo_unpack, dim3(2 * c->num_sms, 2), dim3(256), (const uint32_t*)c->cell_start,
         halo_side(c, true), c->rv, (const uint32_t*)(c->d_xcount + 2), P, L, U, S1, S2, c->d_err, step);
}

void issue_sort(crm_t* c, long long step, uint32_t drop_mask);
void issue_bce(crm_t* c, int stage, float dt, long long step, int store_all);
void issue_rates(crm_t* c, int stage, float dt, long long step);
void issue_rates_range(crm_t* c, int stage, float dt, long long step, long long first, long long count);
void issue_body_partial(crm_t* c);
void issue_body_finish(crm_t* c);

// ---------------------------------------------------------------------------------------
// The phases of one slab step (each ends with posts; the transport flushes between phases).  No
// phase reads the device: the local count is the device word d_slab[0], slot ranges of planes come
// from cellStart inside the kernels, and every transfer has a fixed size (the pack buffers whole),
// so a slab step is one fixed launch sequence per (buffer parity, rebuild) and is replayed from a
// CUDA graph (run_slab_step / crm_group_step).
int slab_phase(crm_t* c, int k, float dt, long long step) {
  static const char* kNames[10] = {"slab P0 pack", "slab P1 append", "slab P2", "slab P3 reuse halo",
                                   "slab P4 sort + BCE(y_n)", "slab P5 rates A boundary", "slab P6 rates A interior",
                                   "slab P7 BCE(y_mid)", "slab P8 rates B", "slab P9 bodies"};
  NvtxRange range(kNames[k < 10 ? k : 9]);
  switch (k) {
    case 0: {   // rebuild: one pass packs emigrants and boundary planes per side (no sort here)
      // Alg. 2: between rebuilds the slots, ghost sets and lists stay; only values move (phase 3)
      c->slab_rebuild = !c->lists_valid || (step >= 0 && (step % c->ps_freq) == 0);
      launch(c, KID_STEP, k_step_begin, dim3(1), dim3(1), c->d_err, step);
      if (!c->slab_rebuild) return CRM_OK;
      const int y = c->cur;
      CK(cudaMemsetAsync(c->pk.cnt, 0, 16, c->stream));
      launch(c, KID_SLAB, k_slab_pack, dim3(8 * c->num_sms), dim3(256), (int)c->ncap, (const float4*)c->P[y],
             (const float4*)c->L[y], c->U[y], (const float4*)c->S1[y], (const float2*)c->S2[y],
             (const uint32_t*)c->ids[y], c->grid, c->x_lo, c->x_hi, c->rank > 0 ? 1 : 0,
             c->rank < c->world - 1 ? 1 : 0, c->pk, c->d_err, step, (const uint32_t*)c->d_slab);
      // counts and the whole pack buffers (E then G of each side): the receiver places them by count
      const size_t pc = (size_t)c->pk.cap_e + c->pk.cap_g;
      for (int d = 0; d < 2; ++d) {
        const int peer = d == 0 ? c->rank - 1 : c->rank + 1;
        post(c, peer, true, c->pk.cnt + 2 * d, 8);
        post_buf(c, peer, true, c->pk, d, pc, true);
        post(c, peer, false, c->rv.cnt + 2 * d, 8);
        post_buf(c, peer, false, c->rv, d, pc, true);
      }
      return CRM_OK;
    }
    case 1: {   // rebuild: immigrants (checked to sit in the boundary plane) and ghosts appended
      if (!c->slab_rebuild) return CRM_OK;
      const int y = c->cur;
      launch(c, KID_SLAB, k_slab_counts, dim3(1), dim3(1), c->d_slab, (const uint32_t*)c->rv.cnt, c->rank > 0 ? 1 : 0,
             c->rank < c->world - 1 ? 1 : 0, c->pk.cap_e, c->pk.cap_g, (uint32_t)c->ncap, c->d_err, step);
      launch(c, KID_SLAB, k_slab_append, dim3(2 * c->num_sms, 2), dim3(256),
             (const uint32_t*)c->d_slab, c->rv, c->P[y], c->L[y], c->U[y], c->S1[y], c->S2[y], c->ids[y], c->grid,
             c->x_lo, c->x_hi, c->d_err, step);
      return CRM_OK;
    }
    case 2:
      return CRM_OK;
    case 3: {   // Alg. 2 reuse step: the ghost planes' y_n refreshed in place
      if (c->slab_rebuild) return CRM_OK;
      const int y = c->cur;
      halo_pack(c, c->P[y], c->L[y], c->U[y], c->S1[y], c->S2[y], step);
      return CRM_OK;
    }
    case 4: {   // the one sort of a rebuild (ghosts in, emigrants and old ghosts out); BCE at y_n; E4
      if (c->slab_rebuild) {
        issue_sort(c, step, TAG_DROP);
        // the new local count: the dropped particles sorted behind cell M
        launch(c, KID_SLAB, k_copy_u32, dim3(1), dim3(1), c->d_slab, (const uint32_t*)(c->cell_start + c->grid.M));
      } else {
        const int y0 = c->cur;
        halo_unpack(c, c->P[y0], c->L[y0], c->U[y0], c->S1[y0], c->S2[y0], step);
      }
      c->ph.build_lists = c->slab_rebuild ? 1 : 0;
      c->lists_valid = true;
      issue_bce(c, 0, dt, step, 0);
      const int y = c->cur;
      halo_pack(c, c->P[y], c->L[y], c->U[y], c->S1[y], c->S2[y], step);
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
        const int y = c->cur;
        halo_unpack(c, c->P[y], c->L[y], c->U[y], c->S1[y], c->S2[y], step);   // E4 -> ghost planes
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
        halo_unpack(c, c->Pm, c->Lm, c->Um, c->S1m, c->S2m, step);   // E5 -> ghost planes of y_mid
        issue_bce(c, 1, dt, step, 0);
      }
      halo_pack(c, c->Pm, c->Lm, c->Um, c->S1m, c->S2m, step);
      return CRM_OK;
    }
    case 8:   // rates + full step; moving bodies: this slab's partial loads to every other slab
      wait_comm(c);
      halo_unpack(c, c->Pm, c->Lm, c->Um, c->S1m, c->S2m, step);   // E7 -> ghost planes of y_mid
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
