// crm.cu — libcrm.so: the C-ABI of include/crm.h and the host orchestration of one step.
//
// One crm_step(dt, n) issues, per step, on the context's stream:
//   memset counts | k_bin | scan (k_scan_tiles, k_scan_add) | k_scatter | k_reorder |
//   k_filter_t (Alg. 1 lists, rebuild steps) | k_bce_t<0> (extrapolation) | k_rates_t<0> (rates + half step) |
//   [k_markers_place(mid)] | k_bce_t<1> | k_rates_t<1> (rates + full step + return map) |
//   [k_body_update | k_body_poses | k_markers_place]
// and synchronises once at the end to read the device error latch.  With world > 1 the same
// kernels run per slab, interleaved with halo exchanges (dist.cuh).
#include "context.cuh"
#include "dist.cuh"

namespace {

// exclusive scan out[0..n] (out[n] = total) of in[0..n) using preallocated level buffers
void scan_u32(crm_t* c, const uint32_t* in, uint32_t* out, long long n, int level) {
  const long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  launch(c, KID_SCAN, k_scan_tiles, dim3((unsigned)tiles), dim3(SCAN_BS), in, out, c->scan_sums[level], n);
  if (tiles == 1) {
    launch(c, KID_COPY, k_copy_u32, dim3(1), dim3(1), out + n, (const uint32_t*)c->scan_sums[level]);
    return;
  }
  scan_u32(c, c->scan_sums[level], c->scan_sums_x[level], tiles, level + 1);
  launch(c, KID_SCAN_ADD, k_scan_add, dim3(blocks(n, 256)), dim3(256), out, (const uint32_t*)c->scan_sums_x[level], n);
  launch(c, KID_COPY, k_copy_u32, dim3(1), dim3(1), out + n, (const uint32_t*)(c->scan_sums_x[level] + tiles));
}

int alloc_debug(crm_t* c) {
  if (c->dbg.drho[0]) return CRM_OK;
  const size_t n = (size_t)c->ncap;
  int r = 0;
  for (int s = 0; s < 2; ++s) {
    r |= dalloc(c, &c->dbg.drho[s], n); r |= dalloc(c, &c->dbg.acc[s], n);
    r |= dalloc(c, &c->dbg.ds1[s], n); r |= dalloc(c, &c->dbg.ds2[s], n);
    r |= dalloc(c, &c->dbg.bu[s], n); r |= dalloc(c, &c->dbg.bs1[s], n); r |= dalloc(c, &c->dbg.bs2[s], n);
  }
  r |= dalloc(c, &c->dbg_ids, n);
  return r ? CRM_E_OOM : CRM_OK;
}

void set_attrs(crm_t* c) {
  if (c->attrs_set) return;
  const int sm = (int)sizeof(TileSmem);
  cudaFuncSetAttribute(k_filter_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FilterSmem));
  // the attribute belongs to the function, not the context: the largest rr buffer (cap <= 255)
  cudaFuncSetAttribute(k_bce_t<0, KER_CUBIC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_bce_t<1, KER_CUBIC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_rates_t<0, KER_CUBIC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_rates_t<1, KER_CUBIC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_bce_t<0, KER_WENDLAND>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_bce_t<1, KER_WENDLAND>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_rates_t<0, KER_WENDLAND>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_rates_t<1, KER_WENDLAND>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  c->attrs_set = true;
}

int commit(crm_t* c) {
  if (c->committed) return CRM_OK;
  if (c->n <= 0) return fail(c, CRM_E_STATE, "no particles added");
  if (c->n >= (int64_t)0xffffffffLL) return fail(c, CRM_E_INVALID, "too many particles for 32-bit indices");
  // ---- which particles are local (slab mode: the owned planes only; ghosts come with step 1)
  std::vector<uint32_t> owned;
  if (c->slab) {
    const int Nx = c->grid.dims[0];
    std::vector<int64_t> counts(Nx, 0);
    std::vector<int> plane(c->n);
    for (int64_t i = 0; i < c->n; ++i) {
      const int p = host_plane(c->grid, c->hP[i].x);
      if (p < 0 || p >= Nx) return fail(c, CRM_E_DOMAIN, "particle id " + std::to_string(i) + " outside the grid box");
      plane[i] = p;
      counts[p]++;
    }
    std::vector<int> bounds(c->world + 1);
    if (slab_partition(counts.data(), Nx, c->world, TX, bounds.data()))
      return fail(c, CRM_E_INVALID, "grid too narrow for the number of slabs");
    c->x_lo = bounds[c->rank];
    c->x_hi = bounds[c->rank + 1];
    int64_t maxp = 0, own = 0;
    for (int p = 0; p < Nx; ++p) maxp = std::max(maxp, counts[p]);
    for (int p = c->x_lo; p < c->x_hi; ++p) own += counts[p];
    owned.reserve(own);
    for (int64_t i = 0; i < c->n; ++i)
      if (plane[i] >= c->x_lo && plane[i] < c->x_hi) owned.push_back((uint32_t)i);
    c->ncap = own + own / 4 + 6 * maxp + 4096;
  } else {
    c->x_lo = 0;
    c->x_hi = c->grid.dims[0];
    c->ncap = c->n;
  }
  c->nl = c->slab ? (int64_t)owned.size() : c->n;
  c->n_owned = c->nl;
  const size_t n = (size_t)c->ncap;
  int r = 0;
  for (int b = 0; b < 2; ++b) {
    r |= dalloc(c, &c->P[b], n); r |= dalloc(c, &c->L[b], n); r |= dalloc(c, &c->U[b], n);
    r |= dalloc(c, &c->S1[b], n); r |= dalloc(c, &c->S2[b], n); r |= dalloc(c, &c->ids[b], n);
  }
  r |= dalloc(c, &c->Pm, n); r |= dalloc(c, &c->Lm, n); r |= dalloc(c, &c->Um, n); r |= dalloc(c, &c->S1m, n); r |= dalloc(c, &c->S2m, n);
  r |= dalloc(c, &c->key, n); r |= dalloc(c, &c->arrival, n);
  r |= dalloc(c, &c->cell_count, (size_t)c->grid.M + 1); r |= dalloc(c, &c->cell_start, (size_t)c->grid.M + 2);
  r |= dalloc(c, &c->tmp_src, n); r |= dalloc(c, &c->tmp_id, n); r |= dalloc(c, &c->cell_of, n);
  r |= dalloc(c, &c->slot_of_id, (size_t)c->n);
  r |= dalloc(c, &c->list, n * (size_t)c->cap); r |= dalloc(c, &c->nlist, n);
  r |= dalloc(c, &c->d_err, 1);
  r |= dalloc(c, &c->d_mtiles, (size_t)std::max<long long>(num_tiles(c->grid), 1)); r |= dalloc(c, &c->d_mtile_cnt, 1);
  r |= dalloc(c, &c->d_xcount, 8);
  if (c->slab) {   // pack buffers: emigrants (E) and a boundary plane (G) per side
    int64_t maxp = 0;
    {
      std::vector<int64_t> cnt(c->grid.dims[0], 0);
      for (int64_t i = 0; i < c->n; ++i) cnt[host_plane(c->grid, c->hP[i].x)]++;
      for (int64_t v : cnt) maxp = std::max(maxp, v);
    }
    // (fixed-size transfers: the emigrants of one rebuild are a fraction of a plane; the boundary plane
    //  may densify by a quarter before CRM_E_CAPACITY is latched)
    c->pk.cap_e = (uint32_t)(maxp / 2 + 1024);
    c->pk.cap_g = (uint32_t)(maxp + maxp / 4 + 1024);
    if (const char* v = std::getenv("CRM_SLAB_CAP_G")) c->pk.cap_g = (uint32_t)std::max(1, std::atoi(v));   // (tests)
    const size_t pc = (size_t)c->pk.cap_e + c->pk.cap_g;
    for (int d = 0; d < 2; ++d) {
      r |= dalloc(c, &c->pk.P[d], pc); r |= dalloc(c, &c->pk.L[d], pc); r |= dalloc(c, &c->pk.U[d], pc);
      r |= dalloc(c, &c->pk.S1[d], pc); r |= dalloc(c, &c->pk.S2[d], pc); r |= dalloc(c, &c->pk.id[d], pc);
    }
    r |= dalloc(c, &c->pk.cnt, 4);
    c->rv.cap_e = c->pk.cap_e;
    c->rv.cap_g = c->pk.cap_g;
    for (int d = 0; d < 2; ++d) {
      r |= dalloc(c, &c->rv.P[d], pc); r |= dalloc(c, &c->rv.L[d], pc); r |= dalloc(c, &c->rv.U[d], pc);
      r |= dalloc(c, &c->rv.S1[d], pc); r |= dalloc(c, &c->rv.S2[d], pc); r |= dalloc(c, &c->rv.id[d], pc);
    }
    r |= dalloc(c, &c->rv.cnt, 4);
    r |= dalloc(c, &c->d_slab, 16);
  }
  c->acap = (int64_t)n;
  if (!c->boxes.empty()) {   // active domains (Alg. 3)
    r |= dalloc(c, &c->d_boxes, c->boxes.size());
    r |= dalloc(c, &c->d_act, n); r |= dalloc(c, &c->d_act_id, (size_t)c->n);
    r |= dalloc(c, &c->d_actcnt, 3);
    r |= dalloc(c, &c->d_tile_list, (size_t)num_tiles(c->grid)); r |= dalloc(c, &c->d_tile_cnt, 1);
    if (!r) {
      CK(cudaMemcpyAsync(c->d_boxes, c->boxes.data(), c->boxes.size() * sizeof(ActiveBox), cudaMemcpyHostToDevice,
                         c->stream));
      CK(cudaMemsetAsync(c->d_act_id, 0, (size_t)c->n, c->stream));
    }
  }
  if (r) return CRM_E_OOM;
  // tiles over the owned planes
  {
    const long long per_x = (long long)tiles_y(c->grid) * tiles_z(c->grid);
    c->tile_base = (long long)(c->x_lo / TX) * per_x;
    c->ntiles = (long long)((c->x_hi - c->x_lo + TX - 1) / TX) * per_x;
  }
  // scan level buffers (M + 1 entries: the last one counts dropped particles)
  long long len = (long long)c->grid.M + 1;
  while (true) {
    const long long tiles = (len + SCAN_TILE - 1) / SCAN_TILE;
    uint32_t *s = nullptr, *sx = nullptr;
    if (dalloc(c, &s, (size_t)tiles) || dalloc(c, &sx, (size_t)tiles + 1)) return CRM_E_OOM;
    c->scan_sums.push_back(s);
    c->scan_sums_x.push_back(sx);
    if (tiles == 1) break;
    len = tiles;
  }
  CK(cudaMallocHost((void**)&c->h_err, sizeof(ErrLatch)));
  CK(cudaMallocHost((void**)&c->h_pin, 64 * sizeof(uint32_t)));
  // bodies and moving markers
  const int nb = (int)c->bodies.size();
  if (dalloc(c, &c->d_bodies, nb) || dalloc(c, &c->d_pose0, nb) || dalloc(c, &c->d_posem, nb)) return CRM_E_OOM;
  std::vector<uint32_t> mids, mstart;
  std::vector<float4> xl;
  std::vector<int> mb;
  for (int b = 1; b < nb; ++b) {
    if (c->bodies[b].motion == CRM_BODY_FIXED) continue;
    double R[9];
    host_quat_R(c->bodies[b].quat, R);
    mb.push_back(b);
    mstart.push_back((uint32_t)mids.size());
    for (int64_t i = 0; i < c->n; ++i) {
      if (c->hBody[i] != b) continue;
      mids.push_back((uint32_t)i);
      const double d[3] = {c->hP[i].x - c->bodies[b].pos[0], c->hP[i].y - c->bodies[b].pos[1],
                           c->hP[i].z - c->bodies[b].pos[2]};
      xl.push_back(make_float4((float)(R[0] * d[0] + R[3] * d[1] + R[6] * d[2]),
                               (float)(R[1] * d[0] + R[4] * d[1] + R[7] * d[2]),
                               (float)(R[2] * d[0] + R[5] * d[1] + R[8] * d[2]), 0.f));
    }
  }
  mstart.push_back((uint32_t)mids.size());
  c->n_moving_markers = (int)mids.size();
  c->n_moving_bodies = (int)mb.size();
  if (c->n_moving_bodies) {   // (a moving body may carry no markers: an active-box carrier)
    mids.reserve(1); xl.reserve(1);
    if (dalloc(c, &c->d_moving_ids, std::max<size_t>(mids.size(), 1)) || dalloc(c, &c->d_xlocal, std::max<size_t>(xl.size(), 1)) ||
        dalloc(c, &c->d_mstart, mstart.size()) || dalloc(c, &c->d_moving_bodies, mb.size()) ||
        dalloc(c, &c->macc, n) || dalloc(c, &c->d_bpart, (size_t)c->world * mb.size() * 6))
      return CRM_E_OOM;
    if (!mids.empty()) {
      CK(cudaMemcpyAsync(c->d_moving_ids, mids.data(), mids.size() * 4, cudaMemcpyHostToDevice, c->stream));
      CK(cudaMemcpyAsync(c->d_xlocal, xl.data(), xl.size() * 16, cudaMemcpyHostToDevice, c->stream));
    }
    CK(cudaMemcpyAsync(c->d_mstart, mstart.data(), mstart.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_moving_bodies, mb.data(), mb.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->macc, 0, n * sizeof(float4), c->stream));
  }
  CK(cudaMemcpyAsync(c->d_bodies, c->bodies.data(), nb * sizeof(BodyState), cudaMemcpyHostToDevice, c->stream));
  // local state (id order)
  const size_t nl = (size_t)c->nl;
  std::vector<uint32_t> idv(nl);
  if (c->slab) {
    std::vector<float4> P(nl), L(nl), U(nl), S1(nl);
    std::vector<float2> S2(nl);
    for (size_t k = 0; k < nl; ++k) {
      const uint32_t i = owned[k];
      P[k] = c->hP[i]; L[k] = c->hL[i]; U[k] = c->hU[i]; S1[k] = c->hS1[i]; S2[k] = c->hS2[i];
      idv[k] = i;
    }
    CK(cudaMemcpyAsync(c->P[0], P.data(), nl * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->L[0], L.data(), nl * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->U[0], U.data(), nl * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->S1[0], S1.data(), nl * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->S2[0], S2.data(), nl * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    launch(c, KID_SLAB, k_fill_u32, dim3(blocks(c->n, 256)), dim3(256), c->slot_of_id, (long long)c->n, 0xffffffffu);
    std::vector<uint32_t> slots(c->n, 0xffffffffu);
    for (size_t k = 0; k < nl; ++k) slots[owned[k]] = (uint32_t)k;
    CK(cudaMemcpyAsync(c->slot_of_id, slots.data(), (size_t)c->n * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->ids[0], idv.data(), nl * 4, cudaMemcpyHostToDevice, c->stream));
    c->h_pin[40] = (uint32_t)nl;   // the device's local count (the slab step keeps it on the device)
    CK(cudaMemcpyAsync(c->d_slab, c->h_pin + 40, 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  } else {
    for (size_t i = 0; i < nl; ++i) idv[i] = (uint32_t)i;
    CK(cudaMemcpyAsync(c->P[0], c->hP.data(), nl * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->L[0], c->hL.data(), nl * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->U[0], c->hU.data(), nl * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->S1[0], c->hS1.data(), nl * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->S2[0], c->hS2.data(), nl * 8, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->ids[0], idv.data(), nl * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->slot_of_id, idv.data(), nl * 4, cudaMemcpyHostToDevice, c->stream));
  }
  CK(cudaMemsetAsync(c->d_err, 0, sizeof(ErrLatch), c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->cur = 0;
  c->committed = true;
  set_attrs(c);
  c->hP.clear(); c->hP.shrink_to_fit(); c->hL.clear(); c->hL.shrink_to_fit(); c->hU.clear(); c->hU.shrink_to_fit();
  c->hS1.clear(); c->hS1.shrink_to_fit(); c->hS2.clear(); c->hS2.shrink_to_fit();
  // NCCL communicator (collective: every rank commits at the same point)
  if (c->slab && c->has_nccl_id) {
    NcclApi& api = nccl();
    if (!api.ok) return fail(c, CRM_E_COMM, "libnccl.so.2 not found (set CRM_NCCL_LIB)");
    ncclUniqueId id;
    std::memcpy(&id, c->nccl_id, sizeof(id));
    ncclComm_t comm;
    ncclResult_t nr = api.commInitRank(&comm, c->world, id, c->rank);
    if (nr != ncclSuccess) return fail(c, CRM_E_COMM, std::string("ncclCommInitRank: ") + api.errorString(nr));
    c->nccl_comm = comm;
    // the communication stream of the overlapped y_mid halo (dist.cuh, phases 5-7)
    if (cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_boundary, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming) != cudaSuccess)
      return fail(c, CRM_E_CUDA, "communication stream");
  }
  return CRM_OK;
}

}  // namespace

namespace {

// sort phase on the local particles: bin, scan, scatter, reorder; particles whose tag
// matches drop_mask leave the local set.  With active domains (Alg. 3) past t_delay, UpdateActivity
// runs first and Inactive particles go behind the active set, frozen.
void issue_sort(crm_t* c, long long step, uint32_t drop_mask) {
  // slabs: the local count is the device word d_slab[0] (kernels read it; grids span the capacity)
  const uint32_t* dn = c->slab ? (const uint32_t*)c->d_slab : nullptr;
  const int n = (int)(c->slab ? c->ncap : c->nl);
  const int a = c->cur, b = 1 - c->cur;
  const bool act = !c->boxes.empty() && c->t_now > c->t_delay;   // Alg. 3: "if t > t_delay"
  c->active_on = act;
  cudaMemsetAsync(c->cell_count, 0, ((size_t)c->grid.M + 1) * 4, c->stream);
  if (act) {
    cudaMemsetAsync(c->d_actcnt, 0, 3 * sizeof(unsigned long long), c->stream);
    launch(c, KID_ACTIVITY, k_activity, dim3(blocks(n, 256)), dim3(256), n, (const float4*)c->P[a],
           (const float4*)c->L[a], c->U[a], (const uint32_t*)c->ids[a], (const BodyState*)c->d_bodies,
           (const ActiveBox*)c->d_boxes, (int)c->boxes.size(), c->support * (double)c->ker.h, c->d_act, c->d_act_id,
           c->d_actcnt, dn);
  }
  launch(c, KID_BIN, k_bin, dim3(blocks(n, 256)), dim3(256), n, (const float4*)c->P[a], (const float4*)c->U[a],
         (const uint32_t*)c->ids[a], c->grid, drop_mask, (const uint8_t*)(act ? c->d_act : nullptr), c->key,
         c->arrival, c->cell_count, c->d_err, step, dn);
  scan_u32(c, c->cell_count, c->cell_start, (long long)c->grid.M + 1, 0);
  if (act) {   // the tiles the step's kernels run on, and the counts the host sizes arrays from
    cudaMemsetAsync(c->d_tile_cnt, 0, 4, c->stream);
    launch(c, KID_ACTIVITY, k_tile_list, dim3(blocks(c->ntiles, 256)), dim3(256), c->ntiles, c->tile_base, c->grid,
           (const uint32_t*)c->cell_start, c->d_tile_list, c->d_tile_cnt);
    cudaMemcpyAsync(c->h_pin, c->cell_start + c->grid.M, 4, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(c->h_pin + 1, c->d_tile_cnt, 4, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(c->h_pin + 8, c->d_actcnt, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream);
  }
  launch(c, KID_SCATTER, k_scatter, dim3(blocks(n, 256)), dim3(256), n, (const uint32_t*)c->key,
         (const uint32_t*)c->arrival, (const uint32_t*)c->cell_start, (const uint32_t*)c->ids[a], c->tmp_src, c->tmp_id, dn);
  if (c->slab && n)
    launch(c, KID_SLAB, k_clear_slots, dim3(blocks(n, 256)), dim3(256), n, (const uint32_t*)c->ids[a], c->slot_of_id, dn);
  launch(c, KID_REORDER, k_reorder, dim3(blocks(n, 256)), dim3(256), n, (const uint32_t*)c->tmp_src,
         (const uint32_t*)c->tmp_id, (const uint32_t*)c->key, (const uint32_t*)c->cell_start,
         (const float4*)c->P[a], (const float4*)c->L[a], (const float4*)c->U[a], (const float4*)c->S1[a],
         (const float2*)c->S2[a], c->P[b], c->L[b], c->U[b], c->S1[b], c->S2[b], c->ids[b], c->cell_of, c->slot_of_id,
         c->grid.M, act ? 1 : 0, dn);
  c->cur = b;
}

// the arrays indexed by sorted slot < N_{a+e}: neighbour lists, mid state, marker loads
// (stream-ordered allocator: a resize costs no device synchronisation; the first resize returns
// the commit-time cudaMalloc buffers)
template <typename T>
int aalloc(crm_t* c, T** p, size_t n) {
  if (*p) {
    if (c->acap_async) cudaFreeAsync(*p, c->stream);
    else cudaFree(*p);
  }
  *p = nullptr;
  return cudaMallocAsync((void**)p, n * sizeof(T), c->stream) == cudaSuccess ? 0 : 1;
}

int alloc_active_arrays(crm_t* c, int64_t cap) {
  const size_t n = (size_t)std::max<int64_t>(cap, 1);
  int r = 0;
  r |= aalloc(c, &c->list, n * (size_t)c->cap); r |= aalloc(c, &c->nlist, n);
  r |= aalloc(c, &c->Pm, n); r |= aalloc(c, &c->Lm, n); r |= aalloc(c, &c->Um, n); r |= aalloc(c, &c->S1m, n);
  r |= aalloc(c, &c->S2m, n);
  if (c->n_moving_markers) {
    r |= aalloc(c, &c->macc, n);
    if (!r) cudaMemsetAsync(c->macc, 0, n * sizeof(float4), c->stream);
  }
  c->acap_async = true;
  if (r) return fail(c, CRM_E_OOM, "active-set arrays");
  c->acap = cap;
  return CRM_OK;
}

// Alg. 3 steps 2–3 after a rebuild sort: ComputeActiveCount (read back: the host sizes the arrays)
// and ManageArrayMemory with growth G, shrink threshold S and interval S_I
int active_capacity(crm_t* c, long long step) {
  unsigned long long* hc = reinterpret_cast<unsigned long long*>(c->h_pin + 8);
  if (c->active_on) {   // the copies were queued by issue_sort right after the scan
    CK(cudaStreamSynchronize(c->stream));
    c->n_ae = c->h_pin[0];
    c->n_tiles_act = c->h_pin[1];
    c->n_act = (int64_t)hc[0]; c->n_ext = (int64_t)hc[1]; c->n_inact = (int64_t)hc[2];
  } else {
    c->n_ae = c->nl;
    c->n_act = c->n_ae; c->n_ext = 0; c->n_inact = 0;
  }
  int action = 0;
  const int64_t cap = manage_capacity(c->acap, c->n_ae, step, c->growth, c->shrink, c->shrink_interval, &action);
  c->last_action = action;
  if (cap != c->acap) return alloc_active_arrays(c, cap);
  return CRM_OK;
}

// the rebuild sort of a single-GPU step (+ the active-set bookkeeping of Alg. 3)
int issue_rebuild_sort(crm_t* c, long long step) {
  issue_sort(c, step, 0);
  if (!c->boxes.empty()) return active_capacity(c, step);
  return CRM_OK;
}

// BCE extrapolation: stage 0 at y_n (with the marker filter), stage 1 at y_mid
// the tile grid of a step: every tile, or (active domains) the non-empty ones listed by k_tile_list
inline ListShape list_shape(const crm_t* c) { return ListShape{c->cap, (uint32_t)c->acap}; }
inline long long tile_grid(const crm_t* c) { return c->active_on ? c->n_tiles_act : c->ntiles; }
inline const uint32_t* tile_list(const crm_t* c) { return c->active_on ? c->d_tile_list : nullptr; }

template <int KER>
void issue_bce_k(crm_t* c, int stage, long long step) {
  const int dbg = c->dbg_on ? 1 : 0;
  if (tile_grid(c) == 0) return;
  // persistent: two resident CTAs per SM walk the marker tiles listed by k_filter_t
  const dim3 tg((unsigned)std::min<long long>(tile_grid(c), 2LL * c->num_sms)), tb(BCE_THREADS);
  const size_t sm = sizeof(TileSmem);
  const int y = c->cur;
  if (stage == 0)
    launch_smem(c, KID_BCE_A, k_bce_t<0, KER>, tg, tb, sm, c->grid, c->ph, (const uint32_t*)c->cell_start,
                (const float4*)c->P[y], (const float4*)c->L[y], c->U[y], c->S1[y], c->S2[y], (const uint16_t*)c->list,
                (const uint32_t*)c->nlist, (const Pose*)c->d_pose0, list_shape(c), c->dbg, dbg, c->d_err, step,
                (const uint32_t*)c->d_mtiles, (const uint32_t*)c->d_mtile_cnt);
  else
    launch_smem(c, KID_BCE_B, k_bce_t<1, KER>, tg, tb, sm, c->grid, c->ph, (const uint32_t*)c->cell_start,
                (const float4*)c->Pm, (const float4*)c->Lm, c->Um, c->S1m, c->S2m, (const uint16_t*)c->list,
                (const uint32_t*)c->nlist, (const Pose*)c->d_posem, list_shape(c), c->dbg, dbg, c->d_err, step,
                (const uint32_t*)c->d_mtiles, (const uint32_t*)c->d_mtile_cnt);
}

// Alg. 1 lists of every tile particle (rebuild steps of Alg. 2): fluid particles all neighbours,
// markers their fluid neighbours (all of them with store_all, the debug export)
void issue_filter(crm_t* c, long long step, int store_all) {
  const int y = c->cur;
  cudaMemsetAsync(c->d_mtile_cnt, 0, 4, c->stream);
  if (tile_grid(c) == 0) return;
  launch_smem(c, KID_FILTER, k_filter_t, dim3((unsigned)tile_grid(c)), dim3(FILTER_THREADS), sizeof(FilterSmem),
              c->grid, (const uint32_t*)c->cell_start, (const float4*)c->P[y], (const float4*)c->U[y], c->list,
              c->nlist, (const uint32_t*)c->cell_of, list_shape(c), store_all, c->d_err,
              (const uint32_t*)c->ids[y], step, c->tile_base, tile_list(c), c->d_mtiles, c->d_mtile_cnt,
              c->list_order);
}

void issue_bce(crm_t* c, int stage, float dt, long long step, int store_all) {
  (void)dt;
  if (stage == 0 && c->ph.build_lists) {
    issue_filter(c, step, store_all);
  }
  if (!c->n_bce) return;
  if (c->ker.kernel == CRM_KERNEL_WENDLAND) issue_bce_k<KER_WENDLAND>(c, stage, step);
  else issue_bce_k<KER_CUBIC>(c, stage, step);
}

// rates: stage 0 (fluid filter + rates at y_n -> y_mid), stage 1 (rates at y_mid -> y_{n+1})
// (first, count): a range of the slab's tiles in launch order (slabs overlap the y_mid halo with the
// interior columns); count < 0 = all tiles
template <int KER>
void issue_rates_k(crm_t* c, int stage, float dt, long long step, long long first = 0, long long count = -1) {
  const int y = c->cur;
  const int dbg = c->dbg_on ? 1 : 0;
  if (tile_grid(c) == 0) return;
  if (count == 0) return;
  const dim3 tg((unsigned)(count < 0 ? tile_grid(c) : count)), tb(TILE_THREADS);
  const long long tbase = c->tile_base + (count < 0 ? 0 : first);
  const size_t sm = sizeof(TileSmem);
  if (stage == 0)
    launch_smem(c, KID_RATES_A, k_rates_t<0, KER>, tg, tb, sm, c->grid, c->ph, dt, (const uint32_t*)c->cell_start,
                (const float4*)c->P[y], (const float4*)c->L[y], (const float4*)c->U[y], (const float4*)c->S1[y],
                (const float2*)c->S2[y], c->Pm, c->Lm, c->Um, c->S1m, c->S2m, (const uint16_t*)c->list,
                (const uint32_t*)c->nlist, list_shape(c), c->macc, c->dbg, dbg, c->d_err, (const uint32_t*)c->ids[y], step,
                tbase, count < 0 ? tile_list(c) : nullptr);
  else
    launch_smem(c, KID_RATES_B, k_rates_t<1, KER>, tg, tb, sm, c->grid, c->ph, dt, (const uint32_t*)c->cell_start,
                (const float4*)c->Pm, (const float4*)c->Lm, (const float4*)c->Um, (const float4*)c->S1m,
                (const float2*)c->S2m, c->P[y], c->L[y], c->U[y], c->S1[y], c->S2[y], (const uint16_t*)c->list,
                (const uint32_t*)c->nlist, list_shape(c), c->macc, c->dbg, dbg, c->d_err, (const uint32_t*)c->ids[y], step,
                tbase, count < 0 ? tile_list(c) : nullptr);
}

void issue_rates(crm_t* c, int stage, float dt, long long step) {
  if (c->ker.kernel == CRM_KERNEL_WENDLAND) issue_rates_k<KER_WENDLAND>(c, stage, dt, step);
  else issue_rates_k<KER_CUBIC>(c, stage, dt, step);
}

void issue_rates_range(crm_t* c, int stage, float dt, long long step, long long first, long long count) {
  if (c->ker.kernel == CRM_KERNEL_WENDLAND) issue_rates_k<KER_WENDLAND>(c, stage, dt, step, first, count);
  else issue_rates_k<KER_CUBIC>(c, stage, dt, step, first, count);
}

// one RK2 step on one GPU (everything on the stream, no host sync)
// moving bodies: this rank's partial loads into its block of d_bpart (A13)
void issue_body_partial(crm_t* c) {
  const double dt = c->dt_d;   // the caller's fp64 step (the fluid kernels take it as fp32)
  launch(c, KID_BODY, k_body_partial, dim3(c->n_moving_bodies), dim3(BODY_BS), (const int*)c->d_moving_bodies,
         (const uint32_t*)c->d_mstart, (const uint32_t*)c->d_moving_ids, (const uint32_t*)c->slot_of_id,
         (const float4*)c->U[c->cur], (const float4*)c->macc, (const float4*)c->Pm, (const float4*)c->Lm,
         (const BodyState*)c->d_bodies, dt, c->d_bpart + (size_t)c->rank * c->n_moving_bodies * 6);
}

// sum of the ranks' partial loads (rank order), rigid update, poses, markers at t_{n+1}
void issue_body_finish(crm_t* c) {
  const double dt = c->dt_d;
  launch(c, KID_BODY, k_body_integrate, dim3(blocks(c->n_moving_bodies, 64)), dim3(64), c->n_moving_bodies,
         (const int*)c->d_moving_bodies, (const double*)c->d_bpart, c->world, c->d_bodies, dt, c->ker.gravity[0],
         c->ker.gravity[1], c->ker.gravity[2], (const ErrLatch*)c->d_err);
  launch(c, KID_POSES, k_body_poses, dim3(blocks((long long)c->bodies.size(), 64)), dim3(64), (int)c->bodies.size(), (const BodyState*)c->d_bodies,
         0.5 * dt, c->d_pose0, c->d_posem);
  const int y = c->cur;
  if (c->n_moving_markers)
    launch(c, KID_MARKERS, k_markers_place, dim3(blocks(c->n_moving_markers, 128)), dim3(128), c->n_moving_markers,
           (const uint32_t*)c->d_moving_ids, (const float4*)c->d_xlocal, (const uint32_t*)c->slot_of_id,
           (const Pose*)c->d_pose0, c->P[y], c->L[y], c->U[y]);
}

int issue_step(crm_t* c, float dt, long long step) {
  // Alg. 2: rebuild (sort + filtered lists) when t mod ps_freq == 0; otherwise the particles keep
  // their slots and the stored lists are reused without a distance re-check (A17)
  const bool rebuild = !c->lists_valid || (step % c->ps_freq) == 0;
  NvtxRange step_range(rebuild ? "crm step (rebuild)" : "crm step (reuse lists)");
  launch(c, KID_STEP, k_step_begin, dim3(1), dim3(1), c->d_err, step);
  if (rebuild) {
    NvtxRange r_sort("sort (A1-A3)");
    const int r = issue_rebuild_sort(c, step);
    if (r) return r;
  }
  c->ph.build_lists = rebuild ? 1 : 0;
  c->lists_valid = true;
  {
    NvtxRange r_a("filter + BCE + rates, stage A (A4-A7)");
    issue_bce(c, 0, dt, step, 0);
    issue_rates(c, 0, dt, step);
  }
  NvtxRange r_b("BCE + rates + return map, stage B (A5-A9)");
  const int y = c->cur;
  if (c->n_moving_markers)
    launch(c, KID_MARKERS, k_markers_place, dim3(blocks(c->n_moving_markers, 128)), dim3(128), c->n_moving_markers,
           (const uint32_t*)c->d_moving_ids, (const float4*)c->d_xlocal, (const uint32_t*)c->slot_of_id,
           (const Pose*)c->d_posem, c->Pm, c->Lm, c->Um);
  issue_bce(c, 1, dt, step, 0);
  issue_rates(c, 1, dt, step);
  if (c->n_moving_bodies) {
    issue_body_partial(c);
    issue_body_finish(c);
  }
  if (c->dbg_on) cudaMemcpyAsync(c->dbg_ids, c->ids[y], (size_t)c->nl * 4, cudaMemcpyDeviceToDevice, c->stream);
  return CRM_OK;
}

// One single-GPU step, replayed from a CUDA graph when possible.  The launch sequence of a step
// depends only on (buffer parity, rebuild step, dt), so it is captured once per key and replayed;
// per-kernel profiling and debug capture run the kernels one by one instead.  Errors latched
// inside a replayed step report step -1 (the host message names the crm_step call instead).
int run_step(crm_t* c, float dt, long long step) {
  const bool rebuild = !c->lists_valid || (step % c->ps_freq) == 0;
  // (active domains resize arrays between steps from host-read counts: launched one by one)
  if (!c->graphs || c->prof || c->dbg_on || !c->boxes.empty()) return issue_step(c, dt, step);
  const int p = c->cur, q = rebuild ? 1 : 0;
  if (!c->gexec[p][q] || c->gdt[p][q] != c->dt_d) {
    if (c->gexec[p][q]) cudaGraphExecDestroy(c->gexec[p][q]);
    c->gexec[p][q] = nullptr;
    const int64_t l0 = c->launches;
    const bool valid0 = c->lists_valid;
    c->lists_valid = !rebuild;   // make issue_step take the same branch as the key
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int rs = issue_step(c, dt, -1);
    CK(cudaStreamEndCapture(c->stream, &graph));
    if (rs) return rs;
    cudaError_t e = cudaGraphInstantiate(&c->gexec[p][q], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return fail(c, CRM_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    c->gdt[p][q] = c->dt_d;
    c->gcur_after[p][q] = c->cur;
    c->gkernels[p][q] = c->launches - l0;
    c->launches = l0;
    c->cur = p;
    c->lists_valid = valid0;
  }
  CK(cudaGraphLaunch(c->gexec[p][q], c->stream));
  c->graph_replays++;
  c->launches += c->gkernels[p][q];
  c->cur = c->gcur_after[p][q];
  c->lists_valid = true;
  return CRM_OK;
}

// One slab step (NCCL transport), replayed from a CUDA graph like run_step: the phases launch a
// fixed sequence per (buffer parity, rebuild) with fixed-size transfers (dist.cuh), so NCCL's
// point-to-point calls are captured with the kernels and the comm-stream fork/join of the overlapped
// halo.  A capture that fails (a transport that cannot be captured) falls back to eager launches.
int slab_step_eager(crm_t* c, float dt, long long step) {
  for (int k = 0; k < kSlabPhases; ++k) {
    if (int r = slab_phase(c, k, dt, step)) return r;
    if (int r = nccl_flush(c)) return r;
  }
  return CRM_OK;
}
int run_slab_step(crm_t* c, float dt, long long step) {
  const bool rebuild = !c->lists_valid || (step % c->ps_freq) == 0;
  // the first steps run eagerly: NCCL connects its point-to-point channels lazily, at the first
  // transfer to a peer, and that setup (allocations, proxy handshakes) is not a stream operation
  if (c->slab_eager_steps < 2) {
    ++c->slab_eager_steps;
    return slab_step_eager(c, dt, step);
  }
  if (!c->graphs || c->prof || c->dbg_on || c->slab_graph_off) return slab_step_eager(c, dt, step);
  const int p = c->cur, q = rebuild ? 1 : 0;
  if (!c->gexec[p][q] || c->gdt[p][q] != c->dt_d) {
    if (c->gexec[p][q]) cudaGraphExecDestroy(c->gexec[p][q]);
    c->gexec[p][q] = nullptr;
    const int64_t l0 = c->launches;
    const bool valid0 = c->lists_valid;
    c->lists_valid = !rebuild;
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const int rs = slab_step_eager(c, dt, -1);
    const cudaError_t ec = cudaStreamEndCapture(c->stream, &graph);
    cudaError_t ei = cudaErrorUnknown;
    if (!rs && ec == cudaSuccess) ei = cudaGraphInstantiate(&c->gexec[p][q], graph, 0);
    if (graph) cudaGraphDestroy(graph);
    c->gkernels[p][q] = c->launches - l0;
    c->gcur_after[p][q] = c->cur;
    c->launches = l0;
    c->cur = p;
    c->lists_valid = valid0;
    c->posts.clear();
    c->comm_pending = false;
    c->halo_async = false;
    if (rs || ec != cudaSuccess || ei != cudaSuccess) {   // not capturable here: eager from now on
      cudaGetLastError();
      c->gexec[p][q] = nullptr;
      c->slab_graph_off = true;
      return slab_step_eager(c, dt, step);
    }
    c->gdt[p][q] = c->dt_d;
  }
  CK(cudaGraphLaunch(c->gexec[p][q], c->stream));
  c->graph_replays++;
  c->launches += c->gkernels[p][q];
  c->cur = c->gcur_after[p][q];
  c->lists_valid = true;
  return CRM_OK;
}

// One step of in-process slab contexts on one stream (loopback transport), every phase on every
// rank then the matched copies — replayed from one CUDA graph per (buffer parity, rebuild), kept on
// rank 0 (the test bed of the capturable slab step on one GPU).
int group_slab_eager(crm_t** cs, int world, float dt, long long step) {
  for (int k = 0; k < kSlabPhases; ++k) {
    for (int a = 0; a < world; ++a)   // (the ranks step in lockstep: one step number)
      if (int r = slab_phase(cs[a], k, dt, step)) return r;
    if (int r = loopback_flush(cs, world)) return r;
  }
  return CRM_OK;
}
int group_slab_step(crm_t** cs, int world, float dt, long long step) {
  crm_t* c0 = cs[0];
  crm_t* c = c0;   // (error reports of the CK checks)
  const bool rebuild = !c0->lists_valid || (step % c0->ps_freq) == 0;
  bool eager = c0->slab_graph_off;
  for (int a = 0; a < world; ++a) eager = eager || !cs[a]->graphs || cs[a]->prof || cs[a]->dbg_on;
  if (eager) return group_slab_eager(cs, world, dt, step);
  const int p = c0->cur, q = rebuild ? 1 : 0;
  const std::vector<crm_t*> members(cs, cs + world);
  if (members != c0->gmembers) {   // another group of contexts: the captured graphs point at other buffers
    for (int b = 0; b < 2; ++b)
      for (int k = 0; k < 2; ++k) {
        if (c0->ggroup[b][k]) cudaGraphExecDestroy(c0->ggroup[b][k]);
        c0->ggroup[b][k] = nullptr;
      }
    c0->gmembers = members;
  }
  if (!c0->ggroup[p][q] || c0->gdt[p][q] != c0->dt_d) {
    if (c0->ggroup[p][q]) cudaGraphExecDestroy(c0->ggroup[p][q]);
    c0->ggroup[p][q] = nullptr;
    std::vector<int64_t> l0(world);
    std::vector<bool> v0(world);
    for (int a = 0; a < world; ++a) {
      l0[a] = cs[a]->launches;
      v0[a] = cs[a]->lists_valid;
      cs[a]->lists_valid = !rebuild;
    }
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(c0->stream, cudaStreamCaptureModeThreadLocal));
    const int rs = group_slab_eager(cs, world, dt, -1);
    const cudaError_t ec = cudaStreamEndCapture(c0->stream, &graph);
    cudaError_t ei = cudaErrorUnknown;
    if (!rs && ec == cudaSuccess) ei = cudaGraphInstantiate(&c0->ggroup[p][q], graph, 0);
    if (graph) cudaGraphDestroy(graph);
    for (int a = 0; a < world; ++a) {
      cs[a]->gkernels[p][q] = cs[a]->launches - l0[a];
      cs[a]->gcur_after[p][q] = cs[a]->cur;
      cs[a]->launches = l0[a];
      cs[a]->cur = p;
      cs[a]->lists_valid = v0[a];
      cs[a]->posts.clear();
    }
    if (rs || ec != cudaSuccess || ei != cudaSuccess) {
      cudaGetLastError();
      c0->ggroup[p][q] = nullptr;
      c0->slab_graph_off = true;
      return group_slab_eager(cs, world, dt, step);
    }
    c0->gdt[p][q] = c0->dt_d;
  }
  CK(cudaGraphLaunch(c0->ggroup[p][q], c0->stream));
  for (int a = 0; a < world; ++a) {
    cs[a]->launches += cs[a]->gkernels[p][q];
    cs[a]->graph_replays++;
    cs[a]->cur = cs[a]->gcur_after[p][q];
    cs[a]->lists_valid = true;
  }
  return CRM_OK;
}

int read_latch(crm_t* c) {
  CK(cudaMemcpyAsync(c->h_err, c->d_err, sizeof(ErrLatch), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->h_err->code) {
    const ErrLatch e = *c->h_err;
    char buf[256];
    if (e.code == CRM_E_DOMAIN && e.aux == 1)
      snprintf(buf, sizeof buf, "particle id %lld crossed more than one cell plane in step %lld", e.id, e.step);
    else if (e.code == CRM_E_DOMAIN)
      snprintf(buf, sizeof buf, "particle id %lld outside the grid box at step %lld", e.id, e.step);
    else if (e.code == CRM_E_NONFINITE)
      snprintf(buf, sizeof buf, "non-finite state at particle id %lld after step %lld", e.id, e.step);
    else if (e.code == CRM_E_CAPACITY && e.aux == 2)
      snprintf(buf, sizeof buf, "slab pack buffer full (emigrants or boundary plane) at particle id %lld, step %lld",
               e.id, e.step);
    else if (e.code == CRM_E_CAPACITY && e.aux == 3)
      snprintf(buf, sizeof buf, "slab capacity exceeded by the immigrants and ghosts received at step %lld", e.step);
    else if (e.code == CRM_E_CAPACITY && e.aux == 4)
      snprintf(buf, sizeof buf, "slab boundary plane larger than the halo buffer at step %lld", e.step);
    else if (e.code == CRM_E_CAPACITY && e.id < 0)
      snprintf(buf, sizeof buf, "tile window of %lld particles exceeds 16-bit offsets at step %lld", e.aux, e.step);
    else if (e.code == CRM_E_COMM)
      snprintf(buf, sizeof buf, "halo of %lld particles does not match the ghost plane at step %lld", e.aux, e.step);
    else if (e.code == CRM_E_CAPACITY)
      snprintf(buf, sizeof buf, "particle id %lld has %lld neighbours > max_neighbors %d at step %lld", e.id, e.aux,
               c->cap, e.step);
    else
      snprintf(buf, sizeof buf, "device error %d at particle id %lld, step %lld", e.code, e.id, e.step);
    c->err = buf;
    cudaMemsetAsync(c->d_err, 0, sizeof(ErrLatch), c->stream);
    cudaStreamSynchronize(c->stream);
    return e.code;
  }
  return CRM_OK;
}

int ensure_stage(crm_t* c, size_t doubles) {
  if (doubles <= c->stage_cap) return CRM_OK;
  if (c->d_stage) cudaFree(c->d_stage);
  c->d_stage = nullptr;
  c->stage_cap = 0;
  if (dalloc(c, &c->d_stage, doubles)) return CRM_E_OOM;
  c->stage_cap = doubles;
  return CRM_OK;
}

int begin_steps(crm_t* c, double dt) {
  cudaSetDevice(c->device);
  int r = commit(c);
  if (r) return r;
  c->dt_d = dt;
  // the device step counter of the error latch: graph replays advance it from here
  launch(c, KID_STEP, k_latch_set_step, dim3(1), dim3(1), c->d_err, (long long)c->steps_done - 1);
  if (c->poses_dt != dt) {
    launch(c, KID_POSES, k_body_poses, dim3(blocks((long long)c->bodies.size(), 64)), dim3(64), (int)c->bodies.size(), (const BodyState*)c->d_bodies,
           0.5 * dt, c->d_pose0, c->d_posem);
    c->poses_dt = dt;
  }
  return CRM_OK;
}

int end_steps(crm_t* c, int64_t nsteps) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, CRM_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  c->steps_done += nsteps;
  c->dbg_valid = c->dbg_on;
  if (c->slab) {   // the host copies of the slab's counts, once per call (the steps never read them)
    cudaMemcpyAsync(c->h_pin + 41, c->d_slab, 4, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(c->h_pin + 42, c->cell_start + plane_start_index(c, c->x_lo), 4, cudaMemcpyDeviceToHost, c->stream);
    cudaMemcpyAsync(c->h_pin + 43, c->cell_start + plane_start_index(c, c->x_hi), 4, cudaMemcpyDeviceToHost, c->stream);
  }
  int r = read_latch(c);
  if (c->slab && nsteps > 0) {
    c->nl = c->h_pin[41];
    c->n_owned = (int64_t)c->h_pin[43] - (int64_t)c->h_pin[42];
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, CRM_E_CUDA, std::string("step: ") + cudaGetErrorString(e));
  return r;
}

}  // namespace

// =======================================================================================
extern "C" {

const char* crm_strerror(int code) {
  switch (code) {
    case CRM_OK: return "ok";
    case CRM_E_INVALID: return "invalid argument";
    case CRM_E_DOMAIN: return "particle outside the grid box";
    case CRM_E_NONFINITE: return "non-finite state";
    case CRM_E_UNSUPPORTED: return "unsupported option";
    case CRM_E_STATE: return "call not allowed in the current state";
    case CRM_E_OOM: return "out of memory";
    case CRM_E_CUDA: return "CUDA error";
    case CRM_E_COMM: return "communication error";
    case CRM_E_CAPACITY: return "neighbour capacity exceeded";
    default: return "unknown error";
  }
}

const char* crm_kernel_name(int k) { return (k >= 0 && k < KID_COUNT) ? kKernelNames[k] : nullptr; }

int crm_create(const crm_material_t* mat, const crm_kernel_t* ker, const crm_boundary_t* bnd, const crm_dist_t* dist,
               crm_t** out) {
  if (!out) return CRM_E_INVALID;
  *out = nullptr;
  if (!mat || !ker || !bnd) return CRM_E_INVALID;
  const crm_material_t& m = *mat;
  const crm_kernel_t& k = *ker;
  if (!(k.h > 0) || !(k.d0 > 0) || k.h < k.d0 || !(m.rho0 > 0) || !(m.K > 0) || !(m.G > 0) || !(m.mu_s > 0) ||
      m.mu_s > m.mu_2 || !(m.I0 > 0) || m.cohesion < 0 || !(m.grain_d > 0) || k.gamma_a < 0 || k.max_neighbors < 0)
    return CRM_E_INVALID;
  if (k.kernel != CRM_KERNEL_CUBIC && k.kernel != CRM_KERNEL_WENDLAND) return CRM_E_INVALID;
  if (k.support != 0.0 && k.support != 2.0) return CRM_E_UNSUPPORTED;   // both kernels: 2h
  if (bnd->method != CRM_BC_ADAMI) return CRM_E_UNSUPPORTED;
  if (k.ps_freq < 0) return CRM_E_INVALID;
  if (k.visc_mode != CRM_VISC_BILATERAL && k.visc_mode != CRM_VISC_UNILATERAL) return CRM_E_INVALID;
  if (dist && (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world)) return CRM_E_INVALID;
  if (dist && dist->world > 1 && bnd->slab_axis != 0) return CRM_E_UNSUPPORTED;
  if (k.max_neighbors > 0 && ((k.max_neighbors % 8) != 0 || k.max_neighbors > 4096)) return CRM_E_INVALID;
  for (int a = 0; a < 3; ++a)
    if (!(bnd->hi[a] > bnd->lo[a])) return CRM_E_INVALID;
  crm_t* c = new crm();
  c->mat = m;
  c->ker = k;
  c->bnd = *bnd;
  c->support = 2.0;
  const double R = c->support * k.h;
  // grid (B1, B3): dims = ceil((hi - lo) / (support h))
  long long M = 1;
  for (int a = 0; a < 3; ++a) {
    c->grid.lo[a] = (float)bnd->lo[a];
    c->grid.dims[a] = (int)std::ceil((bnd->hi[a] - bnd->lo[a]) / R);
    M *= c->grid.dims[a];
  }
  if (M >= 0xfffffff0LL) {
    delete c;
    return CRM_E_INVALID;
  }
  c->grid.M = (uint32_t)M;
  c->grid.s = (float)R;
  c->grid.R2 = (float)(R * R);
  {
    double amax = 0;
    for (int a = 0; a < 3; ++a) amax = std::max(amax, std::max(std::fabs(bnd->lo[a]), std::fabs(bnd->hi[a])));
    c->grid.margin = (float)(16.0 * amax * std::ldexp(1.0, -23) + 1e-6 * R);
  }
  // physics constants (fp32 copies)
  const double h = k.h;
  c->ph.h = (float)h;
  c->ph.hinv = (float)(1.0 / h);
  c->ph.wnorm = (float)(1.0 / (M_PI * h * h * h));
  c->ph.fnorm = (float)(1.0 / (M_PI * h * h * h * h * h));
  c->ph.R2 = (float)(R * R);
  c->ph.m = (float)(m.rho0 * k.d0 * k.d0 * k.d0);
  c->ph.rho0 = (float)m.rho0;
  const double cs = k.cs > 0 ? k.cs : std::sqrt(m.K / m.rho0);
  c->ph.avc = (float)(k.gamma_a * h * cs);
  c->ph.xi2 = (float)(k.xi2 > 0 ? k.xi2 : 0.01 * h * h);
  for (int a = 0; a < 3; ++a) c->ph.g[a] = (float)k.gravity[a];
  c->ph.K = (float)m.K;
  c->ph.G = (float)m.G;
  c->ph.mu_s = (float)m.mu_s;
  c->ph.mu_2 = (float)m.mu_2;
  c->ph.I0 = (float)m.I0;
  c->ph.coh = (float)m.cohesion;
  c->ph.grain_d = (float)m.grain_d;
  c->ph.unilateral = k.visc_mode == CRM_VISC_UNILATERAL;
  c->ph.build_lists = 1;
  c->ps_freq = k.ps_freq > 0 ? k.ps_freq : 1;
  {
    const double fnorm = 1.0 / (M_PI * h * h * h * h * h);
    c->ph.kin_a = (float)(2.25 * fnorm / h);
    c->ph.kin_b = (float)(-3.0 * fnorm);
    c->ph.kout = (float)(-0.75 * h * fnorm);
    c->ph.c_av = (float)(2.0 * m.rho0 * k.d0 * k.d0 * k.d0 * k.gamma_a * h * cs);
    const double wa = 21.0 / (16.0 * M_PI * h * h * h);
    c->ph.wd_a = (float)wa;
    c->ph.wd_f = (float)(-5.0 * wa / (h * h));
  }
  // neighbour capacity: twice the lattice count of the 2h ball, rounded up to 32
  if (k.max_neighbors > 0) {
    c->cap = k.max_neighbors;
  } else {
    const double ball = 4.0 / 3.0 * M_PI * std::pow(R / k.d0, 3.0);
    c->cap = std::max(32, (int)(32 * std::ceil(2.0 * ball / 32.0)));
  }
  // stored list order (reading A34): bank-group-major by default; CRM_LIST_ORDER=scan keeps
  // the candidate order (measurement and the order-permutation test)
  {
    const char* lo = std::getenv("CRM_LIST_ORDER");
    c->list_order = (lo && std::strcmp(lo, "scan") == 0) ? 0 : 1;
  }
  // distribution
  if (dist && dist->world > 1) {
    c->rank = dist->rank;
    c->world = dist->world;
    c->slab = true;
    if (dist->nccl_id) {
      std::memcpy(c->nccl_id, dist->nccl_id, 128);
      c->has_nccl_id = true;
    }
  }
  // device
  c->device = dist ? dist->device : 0;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= c->device) {
    cudaGetLastError();
    delete c;
    return CRM_E_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, c->device) != cudaSuccess || prop.major != 10 || cudaSetDevice(c->device) != cudaSuccess) {
    delete c;
    return CRM_E_CUDA;
  }
  c->num_sms = prop.multiProcessorCount;
  if (dist && dist->cuda_stream) {
    c->stream = (cudaStream_t)dist->cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return CRM_E_CUDA;
    }
    c->own_stream = true;
  }
  BodyState walls{};   // body 0: static walls
  walls.quat[0] = 1.0;
  walls.motion = CRM_BODY_FIXED;
  c->bodies.push_back(walls);
  *out = c;
  return CRM_OK;
}

void crm_destroy(crm_t* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  // a borrowed stream (dist->cuda_stream, e.g. another in-process slab context's) may already be
  // destroyed by its owner: wait on the device instead of on the stream handle
  if (c->own_stream && c->stream) cudaStreamSynchronize(c->stream);
  else cudaDeviceSynchronize();
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  if (c->nccl_comm && nccl().commDestroy) nccl().commDestroy((ncclComm_t)c->nccl_comm);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_boundary) cudaEventDestroy(c->ev_boundary);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  for (auto& r : c->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b) {
    cudaFree(c->P[b]); cudaFree(c->L[b]); cudaFree(c->U[b]); cudaFree(c->S1[b]); cudaFree(c->S2[b]); cudaFree(c->ids[b]);
    for (int q = 0; q < 2; ++q)
      if (c->gexec[b][q]) cudaGraphExecDestroy(c->gexec[b][q]);
    for (int q = 0; q < 2; ++q)
      if (c->ggroup[b][q]) cudaGraphExecDestroy(c->ggroup[b][q]);
    cudaFree(c->dbg.drho[b]); cudaFree(c->dbg.acc[b]); cudaFree(c->dbg.ds1[b]); cudaFree(c->dbg.ds2[b]);
    cudaFree(c->dbg.bu[b]); cudaFree(c->dbg.bs1[b]); cudaFree(c->dbg.bs2[b]);
  }
  cudaFree(c->Pm); cudaFree(c->Lm); cudaFree(c->Um); cudaFree(c->S1m); cudaFree(c->S2m);
  cudaFree(c->d_boxes); cudaFree(c->d_act); cudaFree(c->d_act_id); cudaFree(c->d_actcnt);
  cudaFree(c->d_tile_list); cudaFree(c->d_tile_cnt); cudaFree(c->d_mtiles); cudaFree(c->d_mtile_cnt);
  cudaFree(c->key); cudaFree(c->arrival); cudaFree(c->cell_count); cudaFree(c->cell_start);
  cudaFree(c->tmp_src); cudaFree(c->tmp_id); cudaFree(c->cell_of); cudaFree(c->slot_of_id);
  cudaFree(c->list); cudaFree(c->nlist); cudaFree(c->list32);
  for (auto p : c->scan_sums) cudaFree(p);
  for (auto p : c->scan_sums_x) cudaFree(p);
  cudaFree(c->d_bodies); cudaFree(c->d_pose0); cudaFree(c->d_posem);
  cudaFree(c->d_moving_ids); cudaFree(c->d_xlocal); cudaFree(c->d_mstart); cudaFree(c->d_moving_bodies);
  for (int d = 0; d < 2; ++d) {
    cudaFree(c->pk.P[d]); cudaFree(c->pk.L[d]); cudaFree(c->pk.U[d]); cudaFree(c->pk.S1[d]); cudaFree(c->pk.S2[d]);
    cudaFree(c->pk.id[d]);
  }
  cudaFree(c->pk.cnt);
  for (int d = 0; d < 2; ++d) {
    cudaFree(c->rv.P[d]); cudaFree(c->rv.L[d]); cudaFree(c->rv.U[d]); cudaFree(c->rv.S1[d]); cudaFree(c->rv.S2[d]);
    cudaFree(c->rv.id[d]);
  }
  cudaFree(c->rv.cnt); cudaFree(c->d_slab);
  cudaFree(c->macc); cudaFree(c->d_bpart); cudaFree(c->d_err); cudaFree(c->d_xcount); cudaFree(c->dbg_ids); cudaFree(c->d_stage);
  if (c->h_err) cudaFreeHost(c->h_err);
  if (c->h_pin) cudaFreeHost(c->h_pin);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int crm_add_fluid(crm_t* c, int64_t n, const double* pos, const double* vel, const double* sig6, int64_t* first_id) {
  if (!c) return CRM_E_INVALID;
  if (c->committed) return fail(c, CRM_E_STATE, "crm_add_fluid after the state went to the device");
  if (n < 0 || (n > 0 && !pos)) return fail(c, CRM_E_INVALID, "bad fluid arrays");
  if (first_id) *first_id = c->n;
  const float tag = u2f(make_tag(0, 0, 0));
  for (int64_t k = 0; k < n; ++k) {
    c->hP.push_back(make_float4((float)pos[3 * k], (float)pos[3 * k + 1], (float)pos[3 * k + 2], (float)c->mat.rho0));
    c->hL.push_back(host_lo(pos + 3 * k));
    const float4 hp = c->hP.back(), hl = c->hL.back();
    const float tg = u2f(tag_with_lo(f2u(tag), hp.x, hp.y, hp.z, hl.x, hl.y, hl.z));
    c->hU.push_back(vel ? make_float4((float)vel[3 * k], (float)vel[3 * k + 1], (float)vel[3 * k + 2], tg)
                        : make_float4(0.f, 0.f, 0.f, tg));
    if (sig6) {
      c->hS1.push_back(make_float4((float)sig6[6 * k], (float)sig6[6 * k + 1], (float)sig6[6 * k + 2], (float)sig6[6 * k + 3]));
      c->hS2.push_back(make_float2((float)sig6[6 * k + 4], (float)sig6[6 * k + 5]));
    } else {
      c->hS1.push_back(make_float4(0.f, 0.f, 0.f, 0.f));
      c->hS2.push_back(make_float2(0.f, 0.f));
    }
    c->hBody.push_back(-1);
  }
  c->n += n;
  c->n_fluid += n;
  return CRM_OK;
}

int crm_add_body(crm_t* c, const crm_body_t* b, int32_t* body_id) {
  if (!c || !b) return CRM_E_INVALID;
  if (c->committed) return fail(c, CRM_E_STATE, "crm_add_body after the state went to the device");
  if (c->bodies.size() >= 0x7f) return fail(c, CRM_E_INVALID, "too many bodies (at most 126 besides the walls)");
  if (b->motion < 0 || b->motion > 2) return fail(c, CRM_E_INVALID, "bad motion");
  if (b->motion == CRM_BODY_FREE && !(b->mass > 0)) return fail(c, CRM_E_INVALID, "free body needs mass > 0");
  const double qn = std::sqrt(b->quat[0] * b->quat[0] + b->quat[1] * b->quat[1] + b->quat[2] * b->quat[2] + b->quat[3] * b->quat[3]);
  if (!(qn > 0)) return fail(c, CRM_E_INVALID, "bad quaternion");
  BodyState s{};
  s.mass = b->mass;
  for (int a = 0; a < 3; ++a) {
    s.inertia[a] = b->inertia[a]; s.pos[a] = b->pos[a]; s.vel[a] = b->vel[a]; s.omega[a] = b->omega[a];
  }
  for (int a = 0; a < 4; ++a) s.quat[a] = b->quat[a] / qn;
  s.motion = b->motion;
  s.dof_mask = b->dof_mask;
  if (body_id) *body_id = (int32_t)c->bodies.size();
  c->bodies.push_back(s);
  return CRM_OK;
}

int crm_add_bce(crm_t* c, int32_t body, int64_t n, const double* pos, int64_t* first_id) {
  if (!c) return CRM_E_INVALID;
  if (c->committed) return fail(c, CRM_E_STATE, "crm_add_bce after the state went to the device");
  if (body < 0 || body >= (int32_t)c->bodies.size() || n < 0 || (n > 0 && !pos))
    return fail(c, CRM_E_INVALID, "bad marker arrays or body");
  if (first_id) *first_id = c->n;
  const bool moving = c->bodies[body].motion != CRM_BODY_FIXED;
  const float tag = u2f(make_tag(1, (uint32_t)body, moving ? 1 : 0));
  for (int64_t k = 0; k < n; ++k) {
    c->hP.push_back(make_float4((float)pos[3 * k], (float)pos[3 * k + 1], (float)pos[3 * k + 2], (float)c->mat.rho0));
    c->hL.push_back(host_lo(pos + 3 * k));
    const float4 hp = c->hP.back(), hl = c->hL.back();
    c->hU.push_back(make_float4(0.f, 0.f, 0.f, u2f(tag_with_lo(f2u(tag), hp.x, hp.y, hp.z, hl.x, hl.y, hl.z))));
    c->hS1.push_back(make_float4(0.f, 0.f, 0.f, 0.f));
    c->hS2.push_back(make_float2(0.f, 0.f));
    c->hBody.push_back(body);
  }
  c->n += n;
  c->n_bce += n;
  return CRM_OK;
}

int64_t crm_count(const crm_t* c, int which) {
  if (!c) return 0;
  switch (which) {
    case CRM_FLUID: return c->n_fluid;
    case CRM_BCE: return c->n_bce;
    case CRM_OWNED: return c->committed ? c->n_owned : (c->slab ? 0 : c->n);
    case CRM_GRAPH_REPLAYS: return c->graph_replays;
    default: return c->n;
  }
}

const char* crm_last_error(const crm_t* c) { return c ? c->err.c_str() : "null context"; }
void* crm_stream(crm_t* c) { return c ? (void*)c->stream : nullptr; }
int64_t crm_launch_count(const crm_t* c) { return c ? c->launches : 0; }

int crm_profile_enable(crm_t* c, int on) {
  if (!c) return CRM_E_INVALID;
  if (!on) prof_flush(c);
  c->prof = on != 0;
  return CRM_OK;
}
int crm_profile_reset(crm_t* c) {
  if (!c) return CRM_E_INVALID;
  prof_flush(c);
  for (int k = 0; k < KID_COUNT; ++k) { c->prof_ms[k] = 0; c->prof_n[k] = 0; }
  return CRM_OK;
}
int crm_profile_read(crm_t* c, int kernel, double* ms, int64_t* nl) {
  if (!c || kernel < 0 || kernel >= KID_COUNT) return CRM_E_INVALID;
  prof_flush(c);
  if (ms) *ms = c->prof_ms[kernel];
  if (nl) *nl = c->prof_n[kernel];
  return CRM_OK;
}
int crm_set_graphs(crm_t* c, int on) {
  if (!c) return CRM_E_INVALID;
  c->graphs = on != 0;
  return CRM_OK;
}

int crm_debug_arm(crm_t* c, int on) {
  if (!c) return CRM_E_INVALID;
  if (c->slab) return fail(c, CRM_E_UNSUPPORTED, "debug capture is single-GPU only");
  int r = commit(c);
  if (r) return r;
  if (on) {
    if (alloc_debug(c)) return fail(c, CRM_E_OOM, "debug buffers");
    const size_t n = (size_t)c->ncap;
    for (int s = 0; s < 2; ++s) {
      cudaMemsetAsync(c->dbg.drho[s], 0, n * 4, c->stream); cudaMemsetAsync(c->dbg.acc[s], 0, n * 16, c->stream);
      cudaMemsetAsync(c->dbg.ds1[s], 0, n * 16, c->stream); cudaMemsetAsync(c->dbg.ds2[s], 0, n * 8, c->stream);
      cudaMemsetAsync(c->dbg.bu[s], 0, n * 16, c->stream); cudaMemsetAsync(c->dbg.bs1[s], 0, n * 16, c->stream);
      cudaMemsetAsync(c->dbg.bs2[s], 0, n * 8, c->stream);
    }
    cudaStreamSynchronize(c->stream);
  }
  c->dbg_on = on != 0;
  return CRM_OK;
}

int crm_step(crm_t* c, double dt, int64_t nsteps) {
  if (!c) return CRM_E_INVALID;
  if (!(dt > 0) || nsteps < 0) return fail(c, CRM_E_INVALID, "dt must be > 0 and nsteps >= 0");
  if (c->slab && !c->has_nccl_id) return fail(c, CRM_E_STATE, "in-process slab contexts step with crm_group_step");
  NvtxRange range("crm_step");
  int r = begin_steps(c, dt);
  if (r) return r;
  if (nsteps == 0) return CRM_OK;
  for (int64_t s = 0; s < nsteps; ++s) {
    const long long step = (long long)(c->steps_done + s);
    if (!c->slab) {
      if ((r = run_step(c, (float)dt, step))) return r;
      c->t_now += dt;
      continue;
    }
    if ((r = run_slab_step(c, (float)dt, step))) return r;
  }
  return end_steps(c, nsteps);
}

int crm_group_step(crm_t** cs, int world, double dt, int64_t nsteps) {
  if (!cs || world < 1) return CRM_E_INVALID;
  NvtxRange range("crm_group_step");
  for (int a = 0; a < world; ++a) {
    if (!cs[a] || cs[a]->world != world || cs[a]->rank != a || cs[a]->has_nccl_id)
      return fail(cs[a], CRM_E_INVALID, "crm_group_step: contexts must be ranks 0..world-1 without an NCCL id");
    if (cs[a]->stream != cs[0]->stream || cs[a]->device != cs[0]->device)
      return fail(cs[a], CRM_E_INVALID, "crm_group_step: contexts must share one device and stream");
  }
  if (!(dt > 0) || nsteps < 0) return fail(cs[0], CRM_E_INVALID, "dt must be > 0 and nsteps >= 0");
  int r;
  for (int a = 0; a < world; ++a)
    if ((r = begin_steps(cs[a], dt))) return r;
  for (int64_t s = 0; s < nsteps; ++s) {
    const long long step0 = (long long)(cs[0]->steps_done + s);
    if (world == 1) {
      if ((r = issue_step(cs[0], (float)dt, step0))) return r;
    } else if ((r = group_slab_step(cs, world, (float)dt, step0))) {
      return r;
    }
    for (int a = 0; a < world; ++a) cs[a]->t_now += dt;
  }
  for (int a = 0; a < world; ++a)
    if ((r = end_steps(cs[a], nsteps))) return r;
  return CRM_OK;
}

int crm_nccl_unique_id(void* out128) {
  if (!out128) return CRM_E_INVALID;
  NcclApi& api = nccl();
  if (!api.ok) return CRM_E_COMM;
  ncclUniqueId id;
  if (api.getUniqueId(&id) != ncclSuccess) return CRM_E_COMM;
  std::memcpy(out128, &id, 128);
  return CRM_OK;
}

int crm_pair_count(crm_t* c, int64_t* fluid_pairs) {
  if (!c || !fluid_pairs) return CRM_E_INVALID;
  if (!c->committed || c->steps_done == 0) return fail(c, CRM_E_STATE, "no step taken yet");
  unsigned long long* d = nullptr;
  CK(cudaMalloc(&d, 8));
  CK(cudaMemsetAsync(d, 0, 8, c->stream));
  const int n = (int)(c->boxes.empty() ? c->nl : c->n_ae);   // slots that have lists
  if (n > 0)
    launch(c, KID_SLAB, k_pair_count, dim3(blocks(n, 256)), dim3(256), n, (const float4*)c->U[c->cur],
           (const uint32_t*)c->nlist, d);
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(d);
  *fluid_pairs = (int64_t)h;
  return CRM_OK;
}

int crm_candidate_count(crm_t* c, int64_t* fluid_candidates, int64_t* marker_candidates) {
  if (!c) return CRM_E_INVALID;
  if (!c->committed || c->steps_done == 0) return fail(c, CRM_E_STATE, "no step taken yet");
  unsigned long long* d = nullptr;
  CK(cudaMalloc(&d, 16));
  CK(cudaMemsetAsync(d, 0, 16, c->stream));
  const int n = (int)(c->boxes.empty() ? c->nl : c->n_ae);
  if (n > 0)
    launch(c, KID_SLAB, k_candidate_count, dim3(blocks(n, 256)), dim3(256), n, c->grid, (const float4*)c->U[c->cur],
           (const uint32_t*)c->cell_of, (const uint32_t*)c->cell_start, d);
  unsigned long long h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(d);
  if (fluid_candidates) *fluid_candidates = (int64_t)h[0];
  if (marker_candidates) *marker_candidates = (int64_t)h[1];
  return CRM_OK;
}

// ---- active domains (Alg. 3) -------------------------------------------------------------
int crm_set_active_box(crm_t* c, int32_t body, const double half_extents[3]) {
  if (!c || !half_extents) return CRM_E_INVALID;
  if (c->committed) return fail(c, CRM_E_STATE, "active boxes are set before the first step");
  if (body < 0 || body >= (int32_t)c->bodies.size()) return fail(c, CRM_E_INVALID, "bad body");
  if (c->world > 1) return fail(c, CRM_E_UNSUPPORTED, "active domains are single-GPU in this build");
  for (int a = 0; a < 3; ++a)
    if (!(half_extents[a] >= 0.0)) return fail(c, CRM_E_INVALID, "half extents must be >= 0");
  ActiveBox bx{};
  for (int a = 0; a < 3; ++a) bx.half[a] = half_extents[a];
  bx.body = body;
  for (auto& e : c->boxes)
    if (e.body == body) { e = bx; return CRM_OK; }
  c->boxes.push_back(bx);
  return CRM_OK;
}

int crm_set_active_policy(crm_t* c, const crm_active_t* p) {
  if (!c || !p) return CRM_E_INVALID;
  if (p->growth < 0 || (p->growth > 0 && p->growth < 1.0) || p->shrink < 0 || p->shrink > 1 || p->shrink_interval < 0)
    return fail(c, CRM_E_INVALID, "growth >= 1, 0 <= shrink <= 1, shrink_interval >= 0");
  c->t_delay = p->t_delay;
  c->growth = p->growth > 0 ? p->growth : 1.2;
  c->shrink = p->shrink > 0 ? p->shrink : 0.75;
  c->shrink_interval = p->shrink_interval > 0 ? p->shrink_interval : 50;
  return CRM_OK;
}

int crm_active_stats(const crm_t* c, int64_t out[6]) {
  if (!c || !out) return CRM_E_INVALID;
  out[0] = c->n_act; out[1] = c->n_ext; out[2] = c->n_inact;
  out[3] = c->n_ae; out[4] = c->acap; out[5] = c->last_action;
  return CRM_OK;
}

int64_t crm_manage_capacity(int64_t capacity, int64_t required, int64_t step, double growth, double shrink,
                            int shrink_interval, int* action) {
  return manage_capacity(capacity, required, step, growth, shrink, shrink_interval, action);
}

int crm_debug_activity(crm_t* c, uint8_t* flags_by_id) {
  if (!c || !flags_by_id) return CRM_E_INVALID;
  if (!c->committed || !c->active_on) {
    std::memset(flags_by_id, 0, (size_t)c->n);
    return CRM_OK;
  }
  CK(cudaMemcpyAsync(flags_by_id, c->d_act_id, (size_t)c->n, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return CRM_OK;
}

int crm_slab_partition(const int64_t* plane_counts, int nplanes, int world, int align, int* bounds) {
  if (!plane_counts || !bounds) return CRM_E_INVALID;
  return slab_partition(plane_counts, nplanes, world, align, bounds);
}

int crm_get_state(crm_t* c, int64_t first, int64_t count, double* pos, double* vel, double* rho, double* sig6) {
  if (!c) return CRM_E_INVALID;
  cudaSetDevice(c->device);
  int r = commit(c);
  if (r) return r;
  if (first < 0 || count < 0 || first + count > c->n) return fail(c, CRM_E_INVALID, "id range out of bounds");
  if (count == 0) return CRM_OK;
  if (ensure_stage(c, (size_t)count * 13)) return CRM_E_OOM;
  double* dp = c->d_stage;
  double* dv = dp + 3 * count;
  double* dr = dv + 3 * count;
  double* ds = dr + count;
  if (c->slab) CK(cudaMemsetAsync(dp, 0xff, (size_t)count * 13 * 8, c->stream));   // NaN rows: not owned here
  const int y = c->cur;
  launch(c, KID_STATE, k_get_state, dim3(blocks(count, 256)), dim3(256), (long long)first, (long long)count,
         (const uint32_t*)c->slot_of_id, (const float4*)c->P[y], (const float4*)c->L[y], (const float4*)c->U[y],
         (const float4*)c->S1[y], (const float2*)c->S2[y], dp, dv, dr, ds);
  if (pos) CK(cudaMemcpyAsync(pos, dp, count * 3 * 8, cudaMemcpyDeviceToHost, c->stream));
  if (vel) CK(cudaMemcpyAsync(vel, dv, count * 3 * 8, cudaMemcpyDeviceToHost, c->stream));
  if (rho) CK(cudaMemcpyAsync(rho, dr, count * 8, cudaMemcpyDeviceToHost, c->stream));
  if (sig6) CK(cudaMemcpyAsync(sig6, ds, count * 6 * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return CRM_OK;
}

int crm_set_state(crm_t* c, int64_t first, int64_t count, const double* pos, const double* vel, const double* rho,
                  const double* sig6) {
  if (!c) return CRM_E_INVALID;
  cudaSetDevice(c->device);
  int r = commit(c);
  if (r) return r;
  if (first < 0 || count < 0 || first + count > c->n) return fail(c, CRM_E_INVALID, "id range out of bounds");
  if (count == 0) return CRM_OK;
  if (pos && c->n_moving_markers) {
    std::vector<uint32_t> mids(c->n_moving_markers);
    CK(cudaMemcpy(mids.data(), c->d_moving_ids, mids.size() * 4, cudaMemcpyDeviceToHost));
    for (uint32_t id : mids)
      if ((int64_t)id >= first && (int64_t)id < first + count)
        return fail(c, CRM_E_INVALID, "cannot set the position of a moving-body marker");
  }
  if (ensure_stage(c, (size_t)count * 13)) return CRM_E_OOM;
  double* dp = c->d_stage;
  double* dv = dp + 3 * count;
  double* dr = dv + 3 * count;
  double* ds = dr + count;
  if (pos) CK(cudaMemcpyAsync(dp, pos, count * 3 * 8, cudaMemcpyHostToDevice, c->stream));
  if (pos) c->lists_valid = false;   // positions changed: the next step rebuilds the structure
  if (vel) CK(cudaMemcpyAsync(dv, vel, count * 3 * 8, cudaMemcpyHostToDevice, c->stream));
  if (rho) CK(cudaMemcpyAsync(dr, rho, count * 8, cudaMemcpyHostToDevice, c->stream));
  if (sig6) CK(cudaMemcpyAsync(ds, sig6, count * 6 * 8, cudaMemcpyHostToDevice, c->stream));
  const int y = c->cur;
  launch(c, KID_STATE, k_set_state, dim3(blocks(count, 256)), dim3(256), (long long)first, (long long)count,
         (const uint32_t*)c->slot_of_id, c->P[y], c->L[y], c->U[y], c->S1[y], c->S2[y], (const double*)dp, (const double*)dv,
         (const double*)dr, (const double*)ds, pos ? 1 : 0, vel ? 1 : 0, rho ? 1 : 0, sig6 ? 1 : 0);
  CK(cudaStreamSynchronize(c->stream));
  return CRM_OK;
}

int crm_get_body(crm_t* c, int32_t body, crm_body_t* st, double force[3], double torque[3]) {
  if (!c || body < 0 || body >= (int32_t)c->bodies.size()) return CRM_E_INVALID;
  BodyState b = c->bodies[body];
  if (c->committed) {
    CK(cudaMemcpyAsync(&b, c->d_bodies + body, sizeof(BodyState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  if (st) {
    st->mass = b.mass;
    for (int a = 0; a < 3; ++a) {
      st->inertia[a] = b.inertia[a]; st->pos[a] = b.pos[a]; st->vel[a] = b.vel[a]; st->omega[a] = b.omega[a];
    }
    for (int a = 0; a < 4; ++a) st->quat[a] = b.quat[a];
    st->motion = b.motion;
    st->dof_mask = b.dof_mask;
  }
  for (int a = 0; a < 3; ++a) {
    if (force) force[a] = b.force[a];
    if (torque) torque[a] = b.torque[a];
  }
  return CRM_OK;
}

int crm_debug_structure(crm_t* c, uint32_t* cell_by_id, int64_t* sorted_ids, uint32_t* nbr_count_by_id,
                        uint32_t* cell_start, int64_t* n_cells) {
  if (!c) return CRM_E_INVALID;
  if (c->slab) return fail(c, CRM_E_UNSUPPORTED, "debug exports are single-GPU only");
  cudaSetDevice(c->device);
  int r = commit(c);
  if (r) return r;
  if (n_cells) *n_cells = c->grid.M;
  if (!cell_by_id && !sorted_ids && !nbr_count_by_id && !cell_start) return CRM_OK;
  if ((r = issue_rebuild_sort(c, c->steps_done))) return r;
  c->ph.build_lists = 1;
  c->lists_valid = true;
  issue_bce(c, 0, 0.0f, c->steps_done, 1);   // store_all: every list holds all neighbours, |P(i)|
  issue_rates(c, 0, 0.0f, c->steps_done);
  r = read_latch(c);
  if (r) return r;
  const size_t n = (size_t)c->n;
  // with active domains only the active prefix has lists; Inactive particles have no neighbours
  const size_t nv = c->boxes.empty() ? n : (size_t)c->n_ae;
  std::vector<uint32_t> ids(n), cell(n), cnt(n, 0u);
  CK(cudaMemcpy(ids.data(), c->ids[c->cur], n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cell.data(), c->cell_of, n * 4, cudaMemcpyDeviceToHost));
  if (nv) CK(cudaMemcpy(cnt.data(), c->nlist, nv * 4, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < n; ++s) {
    if (cell_by_id) cell_by_id[ids[s]] = cell[s];
    if (sorted_ids) sorted_ids[s] = ids[s];
    if (nbr_count_by_id) nbr_count_by_id[ids[s]] = cnt[s];
  }
  if (cell_start) CK(cudaMemcpy(cell_start, c->cell_start, ((size_t)c->grid.M + 1) * 4, cudaMemcpyDeviceToHost));
  c->lists_valid = false;   // the export built lists off the Alg. 2 schedule: the next step rebuilds
  return CRM_OK;
}

int crm_debug_neighbors(crm_t* c, int64_t* offsets, int64_t* list) {
  if (!c || !offsets) return CRM_E_INVALID;
  if (c->slab) return fail(c, CRM_E_UNSUPPORTED, "debug exports are single-GPU only");
  cudaSetDevice(c->device);
  int r = commit(c);
  if (r) return r;
  if ((r = issue_rebuild_sort(c, c->steps_done))) return r;
  c->ph.build_lists = 1;
  c->lists_valid = true;
  issue_bce(c, 0, 0.0f, c->steps_done, 1);
  issue_rates(c, 0, 0.0f, c->steps_done);
  const size_t n = (size_t)c->n;
  const size_t nv = c->boxes.empty() ? n : (size_t)c->n_ae;   // slots that have lists (Alg. 3)
  if (!c->list32) {
    if (dalloc(c, &c->list32, n * (size_t)c->cap)) return CRM_E_OOM;
    cudaMemsetAsync(c->list32, 0, n * (size_t)c->cap * 4, c->stream);   // rows are copied whole
  }
  if (nv)
    launch(c, KID_DECODE, k_decode_lists, dim3(blocks((long long)nv, 256)), dim3(256), (int)nv, c->grid,
           (const uint32_t*)c->cell_start, (const uint32_t*)c->cell_of, (const uint16_t*)c->list,
           (const uint32_t*)c->nlist, list_shape(c), c->list32, c->tmp_id /* decoded counts (scratch) */);
  r = read_latch(c);
  if (r) return r;
  c->lists_valid = false;   // store_all lists (markers list all neighbours): the next step rebuilds
  std::vector<uint32_t> ids(n), nl(n, 0u);
  CK(cudaMemcpy(ids.data(), c->ids[c->cur], n * 4, cudaMemcpyDeviceToHost));
  if (nv) CK(cudaMemcpy(nl.data(), c->tmp_id, nv * 4, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> cnt_by_id(n);
  for (size_t s = 0; s < n; ++s) cnt_by_id[ids[s]] = nl[s];
  offsets[0] = 0;
  for (size_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + cnt_by_id[i];
  if (!list) return CRM_OK;
  std::vector<uint32_t> L(nv * (size_t)c->cap);
  if (nv) CK(cudaMemcpy(L.data(), c->list32, L.size() * 4, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < nv; ++s) {
    const uint32_t id = ids[s];
    int64_t* row = list + offsets[id];
    for (uint32_t k = 0; k < nl[s]; ++k) row[k] = ids[L[(size_t)k * nv + s]];
    std::sort(row, row + nl[s]);
  }
  return CRM_OK;
}

int crm_debug_rates(crm_t* c, int stage, double* drho, double* acc, double* dsig6) {
  if (!c || stage < 0 || stage > 1) return CRM_E_INVALID;
  if (!c->dbg_valid) return fail(c, CRM_E_STATE, "no armed step recorded");
  const size_t n = (size_t)c->n;
  std::vector<uint32_t> ids(n);
  std::vector<float> dr(n);
  std::vector<float4> a(n), s1(n);
  std::vector<float2> s2(n);
  CK(cudaMemcpy(ids.data(), c->dbg_ids, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(dr.data(), c->dbg.drho[stage], n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(a.data(), c->dbg.acc[stage], n * 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(s1.data(), c->dbg.ds1[stage], n * 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(s2.data(), c->dbg.ds2[stage], n * 8, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < n; ++s) {
    const uint32_t id = ids[s];
    if (drho) drho[id] = dr[s];
    if (acc) { acc[3 * id] = a[s].x; acc[3 * id + 1] = a[s].y; acc[3 * id + 2] = a[s].z; }
    if (dsig6) {
      dsig6[6 * id] = s1[s].x; dsig6[6 * id + 1] = s1[s].y; dsig6[6 * id + 2] = s1[s].z;
      dsig6[6 * id + 3] = s1[s].w; dsig6[6 * id + 4] = s2[s].x; dsig6[6 * id + 5] = s2[s].y;
    }
  }
  return CRM_OK;
}

int crm_debug_bce(crm_t* c, int stage, double* vel, double* sig6) {
  if (!c || stage < 0 || stage > 1) return CRM_E_INVALID;
  if (!c->dbg_valid) return fail(c, CRM_E_STATE, "no armed step recorded");
  const size_t n = (size_t)c->n;
  std::vector<uint32_t> ids(n);
  std::vector<float4> u(n), s1(n);
  std::vector<float2> s2(n);
  CK(cudaMemcpy(ids.data(), c->dbg_ids, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(u.data(), c->dbg.bu[stage], n * 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(s1.data(), c->dbg.bs1[stage], n * 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(s2.data(), c->dbg.bs2[stage], n * 8, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < n; ++s) {
    const uint32_t id = ids[s];
    if (vel) { vel[3 * id] = u[s].x; vel[3 * id + 1] = u[s].y; vel[3 * id + 2] = u[s].z; }
    if (sig6) {
      sig6[6 * id] = s1[s].x; sig6[6 * id + 1] = s1[s].y; sig6[6 * id + 2] = s1[s].z;
      sig6[6 * id + 3] = s1[s].w; sig6[6 * id + 4] = s2[s].x; sig6[6 * id + 5] = s2[s].y;
    }
  }
  return CRM_OK;
}

#ifdef CRM_EXP_TIMING
int crm_exp_timing(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, crmk::g_exp_timing, sizeof(unsigned long long) * (size_t)n) == cudaSuccess ? 0 : -1;
}
int crm_exp_timing_reset() {
  static unsigned long long z[8192 * 6];
  return cudaMemcpyToSymbol(crmk::g_exp_timing, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
}  // extern "C"
