// context.cuh — the opaque crm_t of include/crm.h and host-side helpers (launch, alloc, errors).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/crm.h"
#include "common.cuh"
#include "physics.cuh"
#include "structure.cuh"
#include "tiled.cuh"
#include "filter.cuh"
#include "active.cuh"

// NVTX range of the host-side launch sequence (an nsys / ncu timeline shows the step's phases; a
// no-op without a tool attached; not recorded by replayed graphs, whose kernels show by name)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

using namespace crmk;

namespace {

enum KernelId {
  KID_MARKERS = 0, KID_BIN, KID_SCAN, KID_SCAN_ADD, KID_SCATTER, KID_REORDER,
  KID_BCE_A, KID_RATES_A, KID_BCE_B, KID_RATES_B, KID_BODY, KID_POSES, KID_STATE, KID_COPY, KID_DECODE,
  KID_SLAB, KID_ACTIVITY, KID_FILTER, KID_STEP, KID_COUNT
};
const char* kKernelNames[KID_COUNT] = {"k_markers_place", "k_bin", "k_scan_tiles", "k_scan_add", "k_scatter",
                                       "k_reorder", "k_bce_A", "k_rates_A", "k_bce_B", "k_rates_B",
                                       "k_body_update", "k_body_poses", "k_get_set_state", "k_copy_u32",
                                       "k_decode_lists", "k_slab_util", "k_activity", "k_filter",
                                       "k_step_begin"};

struct ProfRec {
  int kid;
  cudaEvent_t a, b;
};

// one pending point-to-point transfer of an exchange (multi-GPU)
struct Post {
  int peer;
  bool send;
  void* ptr;
  size_t bytes;
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
  cudaStream_t comm_stream = nullptr;   // slabs: halo transfers that overlap interior tiles (NCCL)
  cudaEvent_t ev_boundary = nullptr, ev_comm = nullptr;
  bool comm_pending = false;            // the compute stream must wait for ev_comm
  bool halo_async = false;              // the next NCCL flush goes to comm_stream (phase 5)
  bool own_stream = false;

  // host staging (id order) until the first device use
  std::vector<float4> hP, hL, hU, hS1;
  std::vector<float2> hS2;
  std::vector<int32_t> hBody;   // -1 for fluid
  std::vector<BodyState> bodies;
  int64_t n = 0, n_fluid = 0, n_bce = 0;   // global id space
  int64_t nl = 0;                          // particles in the local arrays (owned + ghosts)
  int64_t ncap = 0;                        // capacity of the local arrays
  int64_t n_owned = 0;
  bool committed = false;
  int64_t steps_done = 0;

  // device state
  // P = (x hi, rho), L = (x lo, 0): compensated positions x = hi + lo
  float4 *P[2] = {nullptr, nullptr}, *L[2] = {nullptr, nullptr}, *U[2] = {nullptr, nullptr};
  float4* S1[2] = {nullptr, nullptr};
  float2* S2[2] = {nullptr, nullptr};
  uint32_t* ids[2] = {nullptr, nullptr};
  int cur = 0;
  float4 *Pm = nullptr, *Lm = nullptr, *Um = nullptr, *S1m = nullptr;
  float2* S2m = nullptr;
  uint32_t *key = nullptr, *arrival = nullptr, *cell_count = nullptr, *cell_start = nullptr;
  uint32_t *tmp_src = nullptr, *tmp_id = nullptr, *cell_of = nullptr, *slot_of_id = nullptr;
  uint16_t* list = nullptr;             // hot-path lists: window offsets, cap per particle
  uint32_t* nlist = nullptr;            // stored entries per slot (|P(i)| for fluid; all with store_all)
  uint32_t* list32 = nullptr;           // debug only: global indices, ELL k-major
  long long ntiles = 0, tile_base = 0;
  bool attrs_set = false;
  std::vector<uint32_t*> scan_sums, scan_sums_x;
  BodyState* d_bodies = nullptr;
  Pose *d_pose0 = nullptr, *d_posem = nullptr;
  uint32_t* d_moving_ids = nullptr;
  float4* d_xlocal = nullptr;
  uint32_t* d_mstart = nullptr;
  int* d_moving_bodies = nullptr;
  int n_moving_markers = 0, n_moving_bodies = 0;
  float4* macc = nullptr;
  double* d_bpart = nullptr;             // partial body loads, world blocks of n_moving_bodies x 6 (rank order)
  ErrLatch* d_err = nullptr;
  ErrLatch* h_err = nullptr;
  Debug dbg{};
  uint32_t* dbg_ids = nullptr;
  bool dbg_on = false, dbg_valid = false;
  double* d_stage = nullptr;
  size_t stage_cap = 0;
  double poses_dt = -1.0;
  bool graphs = true;
  // captured single-GPU steps, keyed by (buffer parity before the step, rebuild step of Alg. 2)
  cudaGraphExec_t gexec[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  double gdt[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  double dt_d = 0.0;                    // the step of the current crm_step call (fp64: body updates)
  int gcur_after[2][2] = {{0, 0}, {0, 0}};
  int64_t gkernels[2][2] = {{0, 0}, {0, 0}};
  cudaGraphExec_t ggroup[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};   // rank 0 of an in-process slab group
  std::vector<crm_t*> gmembers;         // the contexts the group graphs were captured with
  bool slab_graph_off = false;
  int slab_eager_steps = 0;             // NCCL slab steps run eagerly before the first capture
  int64_t graph_replays = 0;            // steps replayed from a captured graph (crm_count CRM_GRAPH_REPLAYS)          // a slab-step capture failed once: eager launches from then on
  int ps_freq = 1;                      // Alg. 2: lists rebuilt when step % ps_freq == 0
  bool lists_valid = false;             // the stored lists/sort match the current slots
  int list_order = 1;                   // stored list order: 1 bank-group-major (filter.cuh), 0 candidate order
  bool slab_rebuild = true;             // this slab step rebuilds (migration, ghosts, sort, lists)

  // multi-GPU slab decomposition along x
  int rank = 0, world = 1;
  bool slab = false;
  int x_lo = 0, x_hi = 0;               // owned cell planes [x_lo, x_hi)
  void* nccl_comm = nullptr;            // ncclComm_t (NCCL transport); NULL = in-process loopback
  unsigned char nccl_id[128] = {0};
  bool has_nccl_id = false;
  std::vector<Post> posts;
  uint32_t* d_xcount = nullptr;         // device words for count exchanges (send[2], recv[2])
  uint32_t* h_pin = nullptr;            // pinned host scratch (plane ranges, counts)
  // per-step slab bookkeeping (slots in the current buffer)
  uint32_t s_lo = 0, s_lo1 = 0, s_hi1 = 0, s_hi = 0;   // starts of planes x_lo, x_lo+1, x_hi-1, x_hi
  uint32_t s_lom1 = 0, s_hip1 = 0;                     // starts of planes x_lo-1 and x_hi+1 (ghost ranges)
  uint32_t pk_n[4] = {0, 0, 0, 0};     // packed at this rebuild: E_left, G_left, E_right, G_right
  uint32_t rv_n[4] = {0, 0, 0, 0};     // received: E / G from the left, E / G from the right
  SlabPack pk{};                       // pack buffers of the slab rebuild (structure.cuh k_slab_pack) and halos
  SlabPack rv{};                       // receive buffers (the neighbours' pk, whole: fixed-capacity transfers)
  uint32_t* d_slab = nullptr;          // device: [0] local count, [1..4] appended segment starts, [5..8] their sizes

  // active domains (Alg. 3): boxes per body, the active-set capacity of
  // the arrays indexed by sorted slot (lists, mid state, marker loads) and its ManageArrayMemory policy
  std::vector<ActiveBox> boxes;
  ActiveBox* d_boxes = nullptr;
  double t_delay = 0.0, growth = 1.2, shrink = 0.75;
  int shrink_interval = 50;
  double t_now = 0.0;                    // sum of the step sizes taken (compared with t_delay)
  bool active_on = false;                // the last rebuild culled inactive particles
  int64_t acap = 0;                      // capacity of the active-set arrays (slots)
  int64_t n_ae = 0, n_act = 0, n_ext = 0, n_inact = 0;
  int last_action = 0;                   // 0 keep, 1 grow, 2 shrink (crm_manage_capacity)
  uint8_t *d_act = nullptr, *d_act_id = nullptr;   // flags by pre-sort slot / by id
  unsigned long long* d_actcnt = nullptr;
  uint32_t *d_tile_list = nullptr, *d_tile_cnt = nullptr;   // non-empty tiles (kernels launch over them)
  uint32_t *d_mtiles = nullptr, *d_mtile_cnt = nullptr;    // tiles holding markers (k_filter_t -> k_bce_t)
  int num_sms = 148;
  long long n_tiles_act = 0;
  bool acap_async = false;               // active-set arrays come from the stream-ordered allocator

  // profiling
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[KID_COUNT] = {0};
  int64_t prof_n[KID_COUNT] = {0};
  int64_t launches = 0;

  std::string err;
};

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

template <typename Kern, typename... Args>
void launch(crm_t* c, int kid, Kern kern, dim3 grid, dim3 block, Args... args) {
  launch_smem(c, kid, kern, grid, block, 0, args...);
}

inline float u2f(uint32_t u) {
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
inline uint32_t f2u(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
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

// B1 binning of one coordinate on the host (x-plane of a position), same IEEE fp32 ops
inline int host_plane(const Grid& g, float x) {
  volatile float t = (x - g.lo[0]);
  volatile float q = t / g.s;
  return (int)std::floor((float)q);
}

// compensation term of an fp64 position: x - (float)x, per axis
inline float4 host_lo(const double* x) {
  return make_float4((float)(x[0] - (double)(float)x[0]), (float)(x[1] - (double)(float)x[1]),
                     (float)(x[2] - (double)(float)x[2]), 0.f);
}

}  // namespace
