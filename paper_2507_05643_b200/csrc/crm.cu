// crm.cu — libcrm.so: the C-ABI of include/crm.h and the host orchestration of one step.
//
// One crm_step(dt, n) issues, per step, on the context's stream:
//   memset counts | k_bin | scan (k_scan_tiles, k_scan_add) | k_scatter | k_reorder |
//   k_bce_t<0> (marker filter + extrapolation) | k_rates_t<0> (fluid filter + rates + half step) |
//   [k_markers_place(mid)] | k_bce_t<1> | k_rates_t<1> (rates + full step + return map) |
//   [k_body_update | k_body_poses | k_markers_place]
// and synchronises once at the end to read the device error latch.  The step sequence can
// be captured once in a CUDA graph per (dt, buffer parity) and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/crm.h"
#include "common.cuh"
#include "physics.cuh"
#include "structure.cuh"
#include "tiled.cuh"

using namespace crmk;

namespace {

enum KernelId {
  KID_MARKERS = 0, KID_BIN, KID_SCAN, KID_SCAN_ADD, KID_SCATTER, KID_REORDER,
  KID_BCE_A, KID_RATES_A, KID_BCE_B, KID_RATES_B, KID_BODY, KID_POSES, KID_STATE, KID_COPY, KID_DECODE,
  KID_COUNT
};
const char* kKernelNames[KID_COUNT] = {"k_markers_place", "k_bin", "k_scan_tiles", "k_scan_add", "k_scatter",
                                       "k_reorder", "k_bce_A", "k_rates_A", "k_bce_B", "k_rates_B",
                                       "k_body_update", "k_body_poses", "k_get_set_state", "k_copy_u32",
                                       "k_decode_lists"};

struct ProfRec {
  int kid;
  cudaEvent_t a, b;
};

}  // namespace

struct crm {
  crm_material_t mat{};
  crm_kernel_t ker{};
  crm_boundary_t bnd{};
  Grid grid{};
  Phys ph{};
  double support = 2.0;
  int cap = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;

  // host staging (id order) until the first device use
  std::vector<float4> hP, hU, hS1;
  std::vector<float2> hS2;
  std::vector<int32_t> hBody;   // -1 for fluid
  std::vector<BodyState> bodies;
  int64_t n = 0, n_fluid = 0, n_bce = 0;
  bool committed = false;
  int64_t steps_done = 0;

  // device state
  float4 *P[2] = {nullptr, nullptr}, *U[2] = {nullptr, nullptr}, *S1[2] = {nullptr, nullptr};
  float2* S2[2] = {nullptr, nullptr};
  uint32_t* ids[2] = {nullptr, nullptr};
  int cur = 0;
  float4 *Pm = nullptr, *Um = nullptr, *S1m = nullptr;
  float2* S2m = nullptr;
  uint32_t *key = nullptr, *arrival = nullptr, *cell_count = nullptr, *cell_start = nullptr;
  uint32_t *tmp_src = nullptr, *tmp_id = nullptr, *cell_of = nullptr, *slot_of_id = nullptr;
  uint16_t* list = nullptr;             // hot-path lists: window offsets, cap per particle
  uint32_t *nlist = nullptr, *count_all = nullptr;
  uint32_t* list32 = nullptr;           // debug only: global indices, ELL k-major
  long long ntiles = 0;
  bool attrs_set = false;
  std::vector<uint32_t*> scan_sums, scan_sums_x;
  std::vector<long long> scan_len;
  BodyState* d_bodies = nullptr;
  Pose *d_pose0 = nullptr, *d_posem = nullptr;
  uint32_t* d_moving_ids = nullptr;
  float4* d_xlocal = nullptr;
  uint32_t* d_mstart = nullptr;
  int* d_moving_bodies = nullptr;
  int n_moving_markers = 0, n_moving_bodies = 0;
  float4* macc = nullptr;
  ErrLatch* d_err = nullptr;
  ErrLatch* h_err = nullptr;
  Debug dbg{};
  uint32_t* dbg_ids = nullptr;
  bool dbg_on = false, dbg_valid = false;
  double* d_stage = nullptr;
  size_t stage_cap = 0;
  double poses_dt = -1.0;

  // graphs
  bool graphs = true;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  double graph_dt[2] = {-1.0, -1.0};
  bool graph_dbg[2] = {false, false};
  long long* d_step = nullptr;

  // profiling
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[KID_COUNT] = {0};
  int64_t prof_n[KID_COUNT] = {0};
  int64_t launches = 0;

  std::string err;
};

// ---------------------------------------------------------------------------------------
namespace {

int fail(crm_t* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      return fail(c, e_ == cudaErrorMemoryAllocation ? CRM_E_OOM : CRM_E_CUDA,            \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                    \
    }                                                                                     \
  } while (0)

cudaEvent_t get_event(crm_t* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_flush(crm_t* c) {
  if (c->recs.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& r : c->recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    c->prof_ms[r.kid] += ms;
    c->prof_n[r.kid] += 1;
    c->ev_pool.push_back(r.a);
    c->ev_pool.push_back(r.b);
  }
  c->recs.clear();
}

template <typename Kern, typename... Args>
void launch(crm_t* c, int kid, Kern kern, dim3 grid, dim3 block, Args... args) {
  if (grid.x == 0) return;
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->prof) {
    a = get_event(c);
    cudaEventRecord(a, c->stream);
  }
  kern<<<grid, block, 0, c->stream>>>(args...);
  c->launches++;
  if (c->prof) {
    b = get_event(c);
    cudaEventRecord(b, c->stream);
    c->recs.push_back({kid, a, b});
    if (c->recs.size() > 4096) prof_flush(c);
  }
}

template <typename Kern, typename... Args>
void launch_smem(crm_t* c, int kid, Kern kern, dim3 grid, dim3 block, size_t smem, Args... args) {
  if (grid.x == 0) return;
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->prof) {
    a = get_event(c);
    cudaEventRecord(a, c->stream);
  }
  kern<<<grid, block, smem, c->stream>>>(args...);
  c->launches++;
  if (c->prof) {
    b = get_event(c);
    cudaEventRecord(b, c->stream);
    c->recs.push_back({kid, a, b});
    if (c->recs.size() > 4096) prof_flush(c);
  }
}

inline float u2f(uint32_t u) {
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

inline unsigned blocks(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

template <typename T>
int dalloc(crm_t* c, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) return fail(c, CRM_E_OOM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
  return CRM_OK;
}

void host_quat_R(const double q[4], double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

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
  const size_t n = (size_t)c->n;
  int r = 0;
  for (int s = 0; s < 2; ++s) {
    r |= dalloc(c, &c->dbg.drho[s], n); r |= dalloc(c, &c->dbg.acc[s], n);
    r |= dalloc(c, &c->dbg.ds1[s], n); r |= dalloc(c, &c->dbg.ds2[s], n);
    r |= dalloc(c, &c->dbg.bu[s], n); r |= dalloc(c, &c->dbg.bs1[s], n); r |= dalloc(c, &c->dbg.bs2[s], n);
  }
  r |= dalloc(c, &c->dbg_ids, n);
  return r ? CRM_E_OOM : CRM_OK;
}

void set_attrs(crm_t* c);

int commit(crm_t* c) {
  if (c->committed) return CRM_OK;
  if (c->n <= 0) return fail(c, CRM_E_STATE, "no particles added");
  if (c->n >= (int64_t)0xffffffffLL) return fail(c, CRM_E_INVALID, "too many particles for 32-bit indices");
  const size_t n = (size_t)c->n;
  int r = 0;
  for (int b = 0; b < 2; ++b) {
    r |= dalloc(c, &c->P[b], n); r |= dalloc(c, &c->U[b], n); r |= dalloc(c, &c->S1[b], n);
    r |= dalloc(c, &c->S2[b], n); r |= dalloc(c, &c->ids[b], n);
  }
  r |= dalloc(c, &c->Pm, n); r |= dalloc(c, &c->Um, n); r |= dalloc(c, &c->S1m, n); r |= dalloc(c, &c->S2m, n);
  r |= dalloc(c, &c->key, n); r |= dalloc(c, &c->arrival, n);
  r |= dalloc(c, &c->cell_count, (size_t)c->grid.M); r |= dalloc(c, &c->cell_start, (size_t)c->grid.M + 1);
  r |= dalloc(c, &c->tmp_src, n); r |= dalloc(c, &c->tmp_id, n); r |= dalloc(c, &c->cell_of, n);
  r |= dalloc(c, &c->slot_of_id, n);
  r |= dalloc(c, &c->list, n * (size_t)c->cap); r |= dalloc(c, &c->nlist, n); r |= dalloc(c, &c->count_all, n);
  c->ntiles = num_tiles(c->grid);
  r |= dalloc(c, &c->d_err, 1);
  r |= dalloc(c, &c->d_step, 1);
  if (r) return CRM_E_OOM;
  // scan level buffers
  long long len = c->grid.M;
  while (true) {
    const long long tiles = (len + SCAN_TILE - 1) / SCAN_TILE;
    uint32_t *s = nullptr, *sx = nullptr;
    if (dalloc(c, &s, (size_t)tiles) || dalloc(c, &sx, (size_t)tiles + 1)) return CRM_E_OOM;
    c->scan_sums.push_back(s);
    c->scan_sums_x.push_back(sx);
    c->scan_len.push_back(len);
    if (tiles == 1) break;
    len = tiles;
  }
  cudaError_t e = cudaMallocHost((void**)&c->h_err, sizeof(ErrLatch));
  if (e != cudaSuccess) return fail(c, CRM_E_OOM, "cudaMallocHost failed");
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
  if (c->n_moving_markers) {
    if (dalloc(c, &c->d_moving_ids, mids.size()) || dalloc(c, &c->d_xlocal, xl.size()) ||
        dalloc(c, &c->d_mstart, mstart.size()) || dalloc(c, &c->d_moving_bodies, mb.size()) ||
        dalloc(c, &c->macc, n))
      return CRM_E_OOM;
    CK(cudaMemcpyAsync(c->d_moving_ids, mids.data(), mids.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_xlocal, xl.data(), xl.size() * 16, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_mstart, mstart.data(), mstart.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_moving_bodies, mb.data(), mb.size() * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->macc, 0, n * sizeof(float4), c->stream));
  }
  CK(cudaMemcpyAsync(c->d_bodies, c->bodies.data(), nb * sizeof(BodyState), cudaMemcpyHostToDevice, c->stream));
  // state, id order
  CK(cudaMemcpyAsync(c->P[0], c->hP.data(), n * 16, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->U[0], c->hU.data(), n * 16, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->S1[0], c->hS1.data(), n * 16, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->S2[0], c->hS2.data(), n * 8, cudaMemcpyHostToDevice, c->stream));
  std::vector<uint32_t> iota(n);
  for (size_t i = 0; i < n; ++i) iota[i] = (uint32_t)i;
  CK(cudaMemcpyAsync(c->ids[0], iota.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->slot_of_id, iota.data(), n * 4, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemsetAsync(c->d_err, 0, sizeof(ErrLatch), c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->cur = 0;
  c->committed = true;
  set_attrs(c);
  c->hP.clear(); c->hP.shrink_to_fit(); c->hU.clear(); c->hU.shrink_to_fit();
  c->hS1.clear(); c->hS1.shrink_to_fit(); c->hS2.clear(); c->hS2.shrink_to_fit();
  return CRM_OK;
}

// sort phase of a step on the current state: bin, scan, scatter, reorder
void issue_sort(crm_t* c, long long step) {
  const int n = (int)c->n;
  const int a = c->cur, b = 1 - c->cur;
  cudaMemsetAsync(c->cell_count, 0, (size_t)c->grid.M * 4, c->stream);
  launch(c, KID_BIN, k_bin, dim3(blocks(n, 256)), dim3(256), n, (const float4*)c->P[a], (const uint32_t*)c->ids[a],
         c->grid, c->key, c->arrival, c->cell_count, c->d_err, step);
  scan_u32(c, c->cell_count, c->cell_start, c->grid.M, 0);
  launch(c, KID_SCATTER, k_scatter, dim3(blocks(n, 256)), dim3(256), n, (const uint32_t*)c->key,
         (const uint32_t*)c->arrival, (const uint32_t*)c->cell_start, (const uint32_t*)c->ids[a], c->tmp_src, c->tmp_id);
  launch(c, KID_REORDER, k_reorder, dim3(blocks(n, 256)), dim3(256), n, (const uint32_t*)c->tmp_src,
         (const uint32_t*)c->tmp_id, (const uint32_t*)c->key, (const uint32_t*)c->cell_start,
         (const float4*)c->P[a], (const float4*)c->U[a], (const float4*)c->S1[a], (const float2*)c->S2[a],
         c->P[b], c->U[b], c->S1[b], c->S2[b], c->ids[b], c->cell_of, c->slot_of_id);
  c->cur = b;
}

void set_attrs(crm_t* c) {
  if (c->attrs_set) return;
  const int sm = (int)sizeof(TileSmem);
  cudaFuncSetAttribute(k_bce_t<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_bce_t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_rates_t<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  cudaFuncSetAttribute(k_rates_t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  c->attrs_set = true;
}

// stage A (filter + BCE + rates at y_n -> y_mid); store_all keeps marker-marker pairs (debug)
void issue_stage_a(crm_t* c, float dt, long long step, int store_all) {
  const int y = c->cur;
  const int dbg = c->dbg_on ? 1 : 0;
  const dim3 tg((unsigned)c->ntiles), tb(TILE_THREADS);
  const size_t sm = sizeof(TileSmem);
  if (c->n_bce)
    launch_smem(c, KID_BCE_A, k_bce_t<0>, tg, tb, sm, c->grid, c->ph, (const uint32_t*)c->cell_start,
                (const float4*)c->P[y], c->U[y], c->S1[y], c->S2[y], c->list, c->nlist, c->count_all,
                (const uint32_t*)c->cell_of, (const Pose*)c->d_pose0, c->cap, store_all, c->dbg, dbg, c->d_err,
                (const uint32_t*)c->ids[y], step);
  launch_smem(c, KID_RATES_A, k_rates_t<0>, tg, tb, sm, c->grid, c->ph, dt, (const uint32_t*)c->cell_start,
              (const float4*)c->P[y], (const float4*)c->U[y], (const float4*)c->S1[y], (const float2*)c->S2[y], c->Pm,
              c->Um, c->S1m, c->S2m, c->list, c->nlist, c->count_all, (const uint32_t*)c->cell_of, c->cap, c->macc,
              c->dbg, dbg, c->d_err, (const uint32_t*)c->ids[y], step);
}

// one RK2 step (everything on the stream, no host sync)
void issue_step(crm_t* c, float dt, long long step) {
  issue_sort(c, step);
  issue_stage_a(c, dt, step, 0);
  const int y = c->cur;
  const int dbg = c->dbg_on ? 1 : 0;
  const dim3 tg((unsigned)c->ntiles), tb(TILE_THREADS);
  const size_t sm = sizeof(TileSmem);
  if (c->n_moving_markers)
    launch(c, KID_MARKERS, k_markers_place, dim3(blocks(c->n_moving_markers, 128)), dim3(128), c->n_moving_markers,
           (const uint32_t*)c->d_moving_ids, (const float4*)c->d_xlocal, (const uint32_t*)c->slot_of_id,
           (const Pose*)c->d_posem, c->Pm, (const float4*)c->Um);
  // ---- stage B at y_mid, same lists
  if (c->n_bce)
    launch_smem(c, KID_BCE_B, k_bce_t<1>, tg, tb, sm, c->grid, c->ph, (const uint32_t*)c->cell_start,
                (const float4*)c->Pm, c->Um, c->S1m, c->S2m, c->list, c->nlist, c->count_all,
                (const uint32_t*)c->cell_of, (const Pose*)c->d_posem, c->cap, 0, c->dbg, dbg, c->d_err,
                (const uint32_t*)c->ids[y], step);
  launch_smem(c, KID_RATES_B, k_rates_t<1>, tg, tb, sm, c->grid, c->ph, dt, (const uint32_t*)c->cell_start,
              (const float4*)c->Pm, (const float4*)c->Um, (const float4*)c->S1m, (const float2*)c->S2m, c->P[y],
              c->U[y], c->S1[y], c->S2[y], c->list, c->nlist, c->count_all, (const uint32_t*)c->cell_of, c->cap,
              c->macc, c->dbg, dbg, c->d_err, (const uint32_t*)c->ids[y], step);
  // ---- bodies
  if (c->n_moving_bodies) {
    launch(c, KID_BODY, k_body_update, dim3(c->n_moving_bodies), dim3(BODY_BS), (const int*)c->d_moving_bodies,
           (const uint32_t*)c->d_mstart, (const uint32_t*)c->d_moving_ids, (const uint32_t*)c->slot_of_id,
           (const float4*)c->macc, (const float4*)c->Pm, c->d_bodies, (double)dt, c->ph.g[0], c->ph.g[1], c->ph.g[2]);
    launch(c, KID_POSES, k_body_poses, dim3(1), dim3(64), (int)c->bodies.size(), (const BodyState*)c->d_bodies,
           0.5 * (double)dt, c->d_pose0, c->d_posem);
    launch(c, KID_MARKERS, k_markers_place, dim3(blocks(c->n_moving_markers, 128)), dim3(128), c->n_moving_markers,
           (const uint32_t*)c->d_moving_ids, (const float4*)c->d_xlocal, (const uint32_t*)c->slot_of_id,
           (const Pose*)c->d_pose0, c->P[y], (const float4*)c->U[y]);
  }
  if (dbg) cudaMemcpyAsync(c->dbg_ids, c->ids[y], (size_t)c->n * 4, cudaMemcpyDeviceToDevice, c->stream);
}

int read_latch(crm_t* c) {
  CK(cudaMemcpyAsync(c->h_err, c->d_err, sizeof(ErrLatch), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->h_err->code) {
    const ErrLatch e = *c->h_err;
    char buf[256];
    if (e.code == CRM_E_DOMAIN)
      snprintf(buf, sizeof buf, "particle id %lld outside the grid box at step %lld", e.id, e.step);
    else if (e.code == CRM_E_NONFINITE)
      snprintf(buf, sizeof buf, "non-finite state at particle id %lld after step %lld", e.id, e.step);
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
  if (k.kernel != CRM_KERNEL_CUBIC || (k.support != 0.0 && k.support != 2.0)) return CRM_E_UNSUPPORTED;
  if (bnd->method != CRM_BC_ADAMI) return CRM_E_UNSUPPORTED;
  if (k.ps_freq > 1) return CRM_E_UNSUPPORTED;
  if (k.ps_freq < 0) return CRM_E_INVALID;
  if (k.visc_mode != CRM_VISC_BILATERAL && k.visc_mode != CRM_VISC_UNILATERAL) return CRM_E_INVALID;
  if (dist && dist->world > 1) return CRM_E_UNSUPPORTED;
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
  if (M >= 0xffffffffLL) {
    delete c;
    return CRM_E_INVALID;
  }
  c->grid.M = (uint32_t)M;
  c->grid.s = (float)R;
  c->grid.R2 = (float)(R * R);
  {
    // pruning slack: 16 ulp of the largest coordinate + 1e-6 of a cell
    double amax = 0;
    for (int a = 0; a < 3; ++a) amax = std::max(amax, std::max(std::fabs(bnd->lo[a]), std::fabs(bnd->hi[a])));
    c->grid.margin = (float)(16.0 * amax * std::ldexp(1.0, -23) + 1e-6 * R);
  }
  // physics constants
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
  {
    const double fnorm = 1.0 / (M_PI * h * h * h * h * h);
    c->ph.kin_a = (float)(2.25 * fnorm / h);
    c->ph.kin_b = (float)(-3.0 * fnorm);
    c->ph.kout = (float)(-0.75 * h * fnorm);
    c->ph.c_av = (float)(2.0 * m.rho0 * k.d0 * k.d0 * k.d0 * k.gamma_a * h * cs);
  }
  // neighbour capacity: twice the lattice count of the 2h ball, rounded up to 32
  if (k.max_neighbors > 0) {
    c->cap = k.max_neighbors;
  } else {
    const double ball = 4.0 / 3.0 * M_PI * std::pow(R / k.d0, 3.0);
    c->cap = std::max(32, (int)(32 * std::ceil(2.0 * ball / 32.0)));
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
  if (dist && dist->cuda_stream) {
    c->stream = (cudaStream_t)dist->cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return CRM_E_CUDA;
    }
    c->own_stream = true;
  }
  // body 0: static walls
  BodyState walls{};
  walls.quat[0] = 1.0;
  walls.motion = CRM_BODY_FIXED;
  c->bodies.push_back(walls);
  *out = c;
  return CRM_OK;
}

void crm_destroy(crm_t* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& r : c->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b) {
    cudaFree(c->P[b]); cudaFree(c->U[b]); cudaFree(c->S1[b]); cudaFree(c->S2[b]); cudaFree(c->ids[b]);
    if (c->gexec[b]) cudaGraphExecDestroy(c->gexec[b]);
    cudaFree(c->dbg.drho[b]); cudaFree(c->dbg.acc[b]); cudaFree(c->dbg.ds1[b]); cudaFree(c->dbg.ds2[b]);
    cudaFree(c->dbg.bu[b]); cudaFree(c->dbg.bs1[b]); cudaFree(c->dbg.bs2[b]);
  }
  cudaFree(c->Pm); cudaFree(c->Um); cudaFree(c->S1m); cudaFree(c->S2m);
  cudaFree(c->key); cudaFree(c->arrival); cudaFree(c->cell_count); cudaFree(c->cell_start);
  cudaFree(c->tmp_src); cudaFree(c->tmp_id); cudaFree(c->cell_of); cudaFree(c->slot_of_id);
  cudaFree(c->list); cudaFree(c->nlist); cudaFree(c->count_all); cudaFree(c->list32);
  for (auto p : c->scan_sums) cudaFree(p);
  for (auto p : c->scan_sums_x) cudaFree(p);
  cudaFree(c->d_bodies); cudaFree(c->d_pose0); cudaFree(c->d_posem);
  cudaFree(c->d_moving_ids); cudaFree(c->d_xlocal); cudaFree(c->d_mstart); cudaFree(c->d_moving_bodies);
  cudaFree(c->macc); cudaFree(c->d_err); cudaFree(c->d_step); cudaFree(c->dbg_ids); cudaFree(c->d_stage);
  if (c->h_err) cudaFreeHost(c->h_err);
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
    c->hU.push_back(vel ? make_float4((float)vel[3 * k], (float)vel[3 * k + 1], (float)vel[3 * k + 2], tag)
                        : make_float4(0.f, 0.f, 0.f, tag));
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
  if (c->bodies.size() >= 0x7fff) return fail(c, CRM_E_INVALID, "too many bodies");
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
    c->hU.push_back(make_float4(0.f, 0.f, 0.f, tag));
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
  int r = commit(c);
  if (r) return r;
  if (on) {
    if (alloc_debug(c)) return fail(c, CRM_E_OOM, "debug buffers");
    const size_t n = (size_t)c->n;
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
  cudaSetDevice(c->device);
  int r = commit(c);
  if (r) return r;
  if (nsteps == 0) return CRM_OK;
  if (c->poses_dt != dt) {
    launch(c, KID_POSES, k_body_poses, dim3(1), dim3(64), (int)c->bodies.size(), (const BodyState*)c->d_bodies,
           0.5 * dt, c->d_pose0, c->d_posem);
    c->poses_dt = dt;
  }
  for (int64_t s = 0; s < nsteps; ++s) {
    issue_step(c, (float)dt, (long long)(c->steps_done + s));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, CRM_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  c->steps_done += nsteps;
  c->dbg_valid = c->dbg_on;
  r = read_latch(c);
  e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, CRM_E_CUDA, std::string("step: ") + cudaGetErrorString(e));
  return r;
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
  const int y = c->cur;
  launch(c, KID_STATE, k_get_state, dim3(blocks(count, 256)), dim3(256), (long long)first, (long long)count,
         (const uint32_t*)c->slot_of_id, (const float4*)c->P[y], (const float4*)c->U[y], (const float4*)c->S1[y],
         (const float2*)c->S2[y], dp, dv, dr, ds);
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
    // positions of moving-body markers are owned by their body
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
  if (vel) CK(cudaMemcpyAsync(dv, vel, count * 3 * 8, cudaMemcpyHostToDevice, c->stream));
  if (rho) CK(cudaMemcpyAsync(dr, rho, count * 8, cudaMemcpyHostToDevice, c->stream));
  if (sig6) CK(cudaMemcpyAsync(ds, sig6, count * 6 * 8, cudaMemcpyHostToDevice, c->stream));
  const int y = c->cur;
  launch(c, KID_STATE, k_set_state, dim3(blocks(count, 256)), dim3(256), (long long)first, (long long)count,
         (const uint32_t*)c->slot_of_id, c->P[y], c->U[y], c->S1[y], c->S2[y], (const double*)dp, (const double*)dv,
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
  cudaSetDevice(c->device);
  int r = commit(c);
  if (r) return r;
  if (n_cells) *n_cells = c->grid.M;
  if (!cell_by_id && !sorted_ids && !nbr_count_by_id && !cell_start) return CRM_OK;
  issue_sort(c, c->steps_done);
  issue_stage_a(c, 0.0f, c->steps_done, 0);
  r = read_latch(c);
  if (r) return r;
  const size_t n = (size_t)c->n;
  std::vector<uint32_t> ids(n), cell(n), cnt(n);
  CK(cudaMemcpy(ids.data(), c->ids[c->cur], n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cell.data(), c->cell_of, n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cnt.data(), c->count_all, n * 4, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < n; ++s) {
    if (cell_by_id) cell_by_id[ids[s]] = cell[s];
    if (sorted_ids) sorted_ids[s] = ids[s];
    if (nbr_count_by_id) nbr_count_by_id[ids[s]] = cnt[s];
  }
  if (cell_start) CK(cudaMemcpy(cell_start, c->cell_start, ((size_t)c->grid.M + 1) * 4, cudaMemcpyDeviceToHost));
  return CRM_OK;
}

int crm_debug_neighbors(crm_t* c, int64_t* offsets, int64_t* list) {
  if (!c || !offsets) return CRM_E_INVALID;
  cudaSetDevice(c->device);
  int r = commit(c);
  if (r) return r;
  issue_sort(c, c->steps_done);
  issue_stage_a(c, 0.0f, c->steps_done, 1);
  const size_t n = (size_t)c->n;
  if (!c->list32 && dalloc(c, &c->list32, n * (size_t)c->cap)) return CRM_E_OOM;
  launch(c, KID_DECODE, k_decode_lists, dim3(blocks((long long)n, 256)), dim3(256), (int)n, c->grid,
         (const uint32_t*)c->cell_start, (const uint32_t*)c->cell_of, (const uint16_t*)c->list,
         (const uint32_t*)c->nlist, c->cap, c->list32);
  r = read_latch(c);
  if (r) return r;
  std::vector<uint32_t> ids(n), nl(n);
  CK(cudaMemcpy(ids.data(), c->ids[c->cur], n * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(nl.data(), c->nlist, n * 4, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> cnt_by_id(n);
  for (size_t s = 0; s < n; ++s) cnt_by_id[ids[s]] = nl[s];
  offsets[0] = 0;
  for (size_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + cnt_by_id[i];
  if (!list) return CRM_OK;
  std::vector<uint32_t> L(n * (size_t)c->cap);
  CK(cudaMemcpy(L.data(), c->list32, L.size() * 4, cudaMemcpyDeviceToHost));
  for (size_t s = 0; s < n; ++s) {
    const uint32_t id = ids[s];
    int64_t* row = list + offsets[id];
    for (uint32_t k = 0; k < nl[s]; ++k) row[k] = ids[L[(size_t)k * n + s]];
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

}  // extern "C"
