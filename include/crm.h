/* include/crm.h — C-ABI of the B200-native CRM SPH particle update (libcrm.so).
 *
 * The library advances the continuum granular model of Chrono::CRM (arXiv 2507.05643,
 * "A Physics-Based Continuum Model for Versatile, Scalable, and Fast Terramechanics
 * Simulation") by explicit RK2 steps on one NVIDIA B200 (sm_100a), entirely in
 * hand-written CUDA kernels.  One call of crm_step(dt, n) performs, n times, the
 * per-step SPH particle update the paper describes:
 *
 *   1. cell binning   c = cx*(Ny*Nz) + cy*Nz + cz, cell size 2h     (reading B3)
 *   2. sort by (cell, id), cellStart (CSR)                          (B4)
 *   3. Alg. 1 neighbour lists, strict |x_i - x_j| < 2h             (B2)
 *   4. Adami BCE extrapolation of u and sigma onto markers          (A11/A12)
 *   5. rates: continuity (Eq. continuity_dis), momentum with the stress divergence
 *      (Eq. momentum_dis) + artificial viscosity (A9), Jaumann stress
 *      rate (Eq. stress_rate_dis, A4–A6)
 *   6. explicit midpoint RK2 on y = [x, u, rho, sigma]
 *   7. mu(I) return map on sigma* after the full step               (A15/A16)
 *   8. loads of moving rigid bodies from their markers, rigid update (A13)
 *
 * "P:n" = line n of the paper text, "A<k>"/"B<k>" = the readings listed in DESIGN.md.
 *
 * Conventions
 *  - SI units.  Host arrays are fp64, row-major: positions/velocities n x 3, stresses n x 6
 *    in the order (xx, yy, zz, xy, xz, yz), tension positive, sigma = -p I + tau.
 *  - Device state is fp32 structure-of-arrays in HBM, in (cell, id) order, owned by the
 *    library.  All input arrays are copied; the caller keeps ownership of every pointer
 *    it passes.  Output buffers are caller-allocated, sized from crm_count().
 *  - Ids are dense and assigned in call order; fluid particles and BCE markers share one
 *    id space.  crm_get_state returns id order (never the internal sorted order).
 *  - Every call returns 0 (CRM_OK) or a negative CRM_E_* code; crm_last_error() then holds a
 *    message naming the particle id and the step where applicable.
 *  - One context per host thread; not re-entrant.  All GPU work of a call is issued on the
 *    context's stream (crm_stream) and the call synchronises with it before returning.
 *  - No CPU fallback: without a usable sm_100 device crm_create returns CRM_E_CUDA.
 */
#ifndef CRM_H
#define CRM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ---- */
#define CRM_OK             0
#define CRM_E_INVALID     -1   /* bad argument: h <= 0, d0 <= 0, h < d0, dt <= 0, mu_s > mu_2, K/G <= 0 ... */
#define CRM_E_DOMAIN      -2   /* a particle left the fixed grid box (reading A19) */
#define CRM_E_NONFINITE   -3   /* non-finite fluid state after a step */
#define CRM_E_UNSUPPORTED -4   /* option not built: Holmes extrapolation, support != 2, active domains on slabs */
#define CRM_E_STATE       -5   /* crm_add_* after the first step, debug data not available */
#define CRM_E_OOM         -6   /* device or host allocation failed */
#define CRM_E_CUDA        -7   /* CUDA runtime error, or no sm_100 device */
#define CRM_E_COMM        -8   /* NCCL error, or a received halo plane whose count differs from the ghost plane's (multi-GPU) */
#define CRM_E_CAPACITY    -9   /* a particle has more neighbours than crm_kernel_t.max_neighbors, or (slabs) the
                                   fixed-capacity emigrant / boundary-plane / slab buffers overflowed */

#define CRM_KERNEL_CUBIC      0   /* Monaghan (1985) M4 cubic spline, support 2h (A1) */
#define CRM_KERNEL_WENDLAND   1   /* quintic Wendland (Wendland 1995, A28): a (1 - q/2)^4 (2q + 1), support 2h */
#define CRM_VISC_BILATERAL    0   /* Eq. artificial_viscosity_bilateral */
#define CRM_VISC_UNILATERAL   1   /* Eq. artificial_viscosity_unilateral: only v_ij . r_ij < 0 */
#define CRM_BC_ADAMI          0   /* Adami velocity extrapolation */
#define CRM_BC_HOLMES         1   /* named in P:469 without a formula: CRM_E_UNSUPPORTED */
#define CRM_BODY_FIXED        0   /* body 0 (the container walls) is FIXED and pre-created */
#define CRM_BODY_FREE         1   /* rigid body moved by the fluid loads (+ gravity), dof_mask applies */
#define CRM_BODY_PRESCRIBED   2   /* constant linear/angular velocity, loads still reported */
#define CRM_FLUID             0
#define CRM_BCE               1
#define CRM_ALL               2
#define CRM_OWNED             3
#define CRM_GRAPH_REPLAYS     4   /* crm_count: steps of this context replayed from a captured CUDA graph */

typedef struct crm crm_t;   /* opaque; owned by the library */

/* Material of the granular continuum: rho0 reference density, K bulk and G shear
 * moduli of the hypo-elastic law (values unstated in the paper: reading A2),
 * mu_s, mu_2, I0 of mu(I), cohesion c, grain diameter d. */
typedef struct {
  double rho0, K, G, mu_s, mu_2, I0, cohesion, grain_d;
} crm_material_t;

/* SPH discretisation (Table tab:sph_params). */
typedef struct {
  int    kernel;          /* CRM_KERNEL_CUBIC | CRM_KERNEL_WENDLAND (other values: CRM_E_INVALID) */
  double d0, h;           /* initial spacing, smoothing length (h >= d0); particle mass m = rho0 d0^3 */
  double support;         /* kernel support factor K = 2; 0 -> 2 */
  int    visc_mode;       /* CRM_VISC_* */
  double gamma_a;         /* artificial viscosity coefficient */
  double xi2;             /* regulariser xi^2 of Eq. 13; <= 0 -> 0.01 h^2 (A10) */
  double cs;              /* speed of sound; <= 0 -> sqrt(K / rho0) (A10) */
  int    ps_freq;         /* neighbour-list rebuild period (Alg. 2); 0 -> 1.  With ps_freq > 1
                             the stored lists are permuted into a bank-conflict-avoiding order at each
                             rebuild (same neighbour sets; A34; env CRM_LIST_ORDER=rr|scan
                             overrides the choice at crm_create) */
  double gravity[3];      /* body force per unit mass f_b */
  int    max_neighbors;   /* neighbour-list capacity per particle, a multiple of 8, <= 4096; 0 -> derived from h/d0 */
} crm_kernel_t;

/* Boundary handling and the fixed grid box. */
typedef struct {
  int    method;          /* CRM_BC_ADAMI */
  int    n_layers;        /* informational: 0 -> ceil(support h / d0) */
  double lo[3], hi[3];    /* grid box; cells of size support*h tile [lo, lo + ceil((hi-lo)/(support h)) * support h) */
  int    slab_axis;       /* multi-GPU slab axis: 0 = x (the only one supported) */
} crm_boundary_t;

/* Distribution (optional; NULL = one GPU, device 0, library-owned stream). */
typedef struct {
  int rank, world, device;
  const void* nccl_id;    /* 128-byte ncclUniqueId shared by all ranks (world > 1) */
  void* cuda_stream;      /* cudaStream_t to issue on; NULL = library creates one */
} crm_dist_t;

/* Rigid body carrying BCE markers.  Body 0 = the static walls. */
typedef struct {
  double mass, inertia[3];        /* inertia: principal moments about the body axes (Euler equations) */
  double pos[3], quat[4];         /* centre of mass, orientation (w, x, y, z) */
  double vel[3], omega[3];
  int    motion;                  /* CRM_BODY_* */
  int    dof_mask;                /* FREE: bit k set = DOF k free (0..2 translation, 3..5 rotation) */
} crm_body_t;

/* Create a context: validates the parameters (CRM_E_INVALID / CRM_E_UNSUPPORTED), selects the
 * device, creates (or adopts) the stream.  *out is NULL on error. */
int  crm_create(const crm_material_t* mat, const crm_kernel_t* ker, const crm_boundary_t* bnd,
                const crm_dist_t* dist /* nullable */, crm_t** out);
void crm_destroy(crm_t* ctx);

/* Append n fluid particles: pos n x 3 (required), vel n x 3 (NULL -> 0), sig6 n x 6 (NULL -> 0).
 * rho starts at rho0.  *first_id receives the id of the first one.  CRM_E_STATE after a step. */
int  crm_add_fluid(crm_t* ctx, int64_t n, const double* pos, const double* vel, const double* sig6,
                   int64_t* first_id);
/* Add a rigid body (returns its index in *body_id; body 0 exists already).  At most 126 bodies besides
   the walls (the body index shares the marker tag word with the position's compensation term);
   more return CRM_E_INVALID. */
int  crm_add_body(crm_t* ctx, const crm_body_t* body, int32_t* body_id);
/* Append n BCE markers attached to `body`, given in world coordinates at the body's initial pose. */
int  crm_add_bce(crm_t* ctx, int32_t body, int64_t n, const double* pos_world, int64_t* first_id);

/* Advance nsteps explicit RK2 steps of size dt (synchronous).  Returns the first error latched
 * on the device (CRM_E_DOMAIN, CRM_E_NONFINITE, CRM_E_CAPACITY) with the id and the step in
 * which it occurred in crm_last_error (a device step counter, also inside replayed CUDA graphs).
 * The steps after the failing one compute nothing: the state is the one the failing step left,
 * and the call returns after nsteps launches with that first error.  With world > 1 and an NCCL id, every rank calls crm_step with the same
 * arguments; ghost planes are exchanged with NCCL point-to-point transfers (CRM_E_COMM).  A step
 * reads nothing back on the host (slabs too: device-resident counts, fixed-size transfers), so
 * with graphs on (the default, crm_set_graphs) each step after the first of its kind is replayed
 * from a captured CUDA graph (slab contexts over NCCL: captured from the third step on, after NCCL
 * has connected its channels); crm_count(ctx, CRM_GRAPH_REPLAYS) counts the replayed steps. */
int  crm_step(crm_t* ctx, double dt, int64_t nsteps);

/* ---- multi-GPU slab decomposition along x ----
 * A context created with crm_dist_t.world > 1 owns the cell planes [x_lo, x_hi) chosen from a
 * prefix sum of per-plane particle counts of the (identical) global crm_add_* input.  Every rank
 * passes the same global arrays; the library keeps its slab.  crm_get_state then fills only the
 * rows of owned ids (other rows are NaN) and crm_count(ctx, CRM_OWNED) counts them.  The
 * debug exports and active domains are single-GPU only in this build (CRM_E_UNSUPPORTED); moving
 * bodies work on slabs: each slab sums the loads of the markers it owns, the partial sums are
 * exchanged and added in rank order, so every rank integrates the same body state. */
/* Step `world` contexts of ranks 0..world-1 living in one process on one device and stream
 * (nccl_id NULL): exchanges become device copies ("loopback"); used to test the decomposition
 * on one GPU.  Owned particles follow bit-identical trajectories to a one-context run.  The ranks'
 * steps (all phases and copies) are captured together as one CUDA graph, kept by ctxs[0]. */
int  crm_group_step(crm_t** ctxs, int world, double dt, int64_t nsteps);
/* 128-byte ncclUniqueId for crm_dist_t.nccl_id (call on one rank, broadcast to the others). */
int  crm_nccl_unique_id(void* out128);
/* Pure host helper: slab boundaries bounds[0..world] (bounds[0] = 0, bounds[world] = nplanes,
 * interior ones multiples of `align`) balancing the per-plane particle counts.  CRM_E_INVALID if
 * nplanes < world * align. */
int  crm_slab_partition(const int64_t* plane_counts, int nplanes, int world, int align, int* bounds);

/* ---- active domains (Alg. 3; readings A29–A31) ----
 * An "active box" is an oriented box of half extents half_extents[3] (m, body frame) at the local
 * origin of `body`, moving with it (body 0 = the fixed container frame).  After t_delay
 * (Alg. 3 "if t > t_delay"), at every neighbour-list rebuild (Alg. 2 period), each particle is
 * flagged: Active inside a box, Extended-Active outside every box but closer than 2h to
 * one, Inactive otherwise; markers of moving bodies are always Active.  Inactive particles take
 * no part in the neighbour search, their state is frozen (crm_get_state still returns it) and the
 * arrays indexed by the active set (neighbour lists, mid-step state) are sized by the
 * ManageArrayMemory policy (growth G, shrink threshold S every S_I steps).  Single-GPU only
 * (CRM_E_UNSUPPORTED with world > 1); set before the first step (CRM_E_STATE after). */
typedef struct {
  double t_delay;        /* s; culling starts once t > t_delay (default 0) */
  double growth;         /* G; 0 -> 1.2 */
  double shrink;         /* S; 0 -> 0.75 */
  int    shrink_interval;/* S_I steps; 0 -> 50 */
} crm_active_t;
int  crm_set_active_box(crm_t* ctx, int32_t body, const double half_extents[3]);
int  crm_set_active_policy(crm_t* ctx, const crm_active_t* policy);
/* out = {N_active, N_extended, N_inactive, N_{a+e}, capacity, last action (0 keep, 1 grow,
 * 2 shrink)} of the last rebuild. */
int  crm_active_stats(const crm_t* ctx, int64_t out[6]);
/* Pure host helper, the ManageArrayMemory policy: new capacity for `required` elements at step
 * `step`; *action = 0 keep, 1 grow (to ceil(required * growth)), 2 shrink (to required). */
int64_t crm_manage_capacity(int64_t capacity, int64_t required, int64_t step, double growth, double shrink,
                            int shrink_interval, int* action);

/* Copy state of ids [first_id, first_id + count) to host fp64 arrays (any pointer may be NULL).
 * For markers: the last extrapolated u and sigma, rho = rho0. */
int  crm_get_state(crm_t* ctx, int64_t first_id, int64_t count, double* pos, double* vel,
                   double* rho, double* sig6);
/* Overwrite state of ids [first_id, first_id + count) from host fp64 arrays (NULL = keep).
 * Positions of markers of moving bodies cannot be set (CRM_E_INVALID). */
int  crm_set_state(crm_t* ctx, int64_t first_id, int64_t count, const double* pos, const double* vel,
                   const double* rho, const double* sig6);
/* Body pose/velocity and the force/torque of the last step (about the centre of mass). */
int  crm_get_body(crm_t* ctx, int32_t body, crm_body_t* state, double force[3], double torque[3]);
int64_t crm_count(const crm_t* ctx, int which /* CRM_FLUID | CRM_BCE | CRM_ALL | CRM_OWNED | CRM_GRAPH_REPLAYS */);
const char* crm_last_error(const crm_t* ctx);
const char* crm_strerror(int code);

/* ---- measurement helpers ---- */
void*   crm_stream(crm_t* ctx);                 /* the cudaStream_t all kernels are issued on */
int64_t crm_launch_count(const crm_t* ctx);     /* kernels launched by this context so far */
/* Per-kernel timing with CUDA events on crm_stream (off by default).  kernel index 0..n-1,
 * name via crm_kernel_name; ms = accumulated device time, launches = launch count. */
int     crm_profile_enable(crm_t* ctx, int on);
int     crm_profile_read(crm_t* ctx, int kernel, double* ms, int64_t* launches);
int     crm_profile_reset(crm_t* ctx);
const char* crm_kernel_name(int kernel);        /* NULL past the last kernel */
/* Use a CUDA graph for the per-step launch sequence (default on). */
int     crm_set_graphs(crm_t* ctx, int on);
/* Number of directed fluid-particle pairs |P(i)| summed over this rank's owned fluid particles,
 * as built by the last step (the work of the rates loops; bench.py roofline).  CRM_E_STATE before
 * the first step. */
int     crm_pair_count(crm_t* ctx, int64_t* fluid_pairs);
/* Alg. 1 candidates of the last structure: for every owned particle, the particles of
 * the 27 cells around its cell minus itself, summed over fluid particles and over markers (the
 * work of the neighbour filter; bench.py roofline).  CRM_E_STATE before the first step. */
int     crm_candidate_count(crm_t* ctx, int64_t* fluid_candidates, int64_t* marker_candidates);

/* ---- test-only exports (parity harness) ---- */
/* Arm/disarm capture of per-step rates and BCE values (costs extra HBM writes). */
int  crm_debug_arm(crm_t* ctx, int on);
/* Structure of the CURRENT state (what the next step builds first): cell id per particle id,
 * the sorted id order, neighbour counts per id (all fluid + BCE neighbours), cellStart (M+1).
 * Any pointer may be NULL; *n_cells receives M.  Both structure exports re-sort the state and
 * rebuild the lists off the Alg. 2 schedule, so the step after an export is a rebuild step
 * (with ps_freq > 1 an inspected run therefore differs from an uninspected one; at ps_freq = 1,
 * where every step rebuilds, it does not). */
int  crm_debug_structure(crm_t* ctx, uint32_t* cell_by_id, int64_t* sorted_ids,
                         uint32_t* nbr_count_by_id, uint32_t* cell_start, int64_t* n_cells);
/* Neighbour sets of the CURRENT state by id, CSR (offsets n+1), rows ascending by id. */
int  crm_debug_neighbors(crm_t* ctx, int64_t* offsets, int64_t* list /* NULL = counts only */);
/* Rates of the last armed step by id: stage 0 = A (at y_n), 1 = B (at y_mid).  Fluid rows:
 * drho, acc, dsigma; rows of moving-body markers: acc only (stage B). */
int  crm_debug_rates(crm_t* ctx, int stage, double* drho, double* acc, double* dsig6);
/* Extrapolated marker velocity and stress of the last armed step's stage, by id. */
int  crm_debug_bce(crm_t* ctx, int stage, double* vel, double* sig6);
/* Activity flags (0 Active, 1 Extended-Active, 2 Inactive) by id of the last rebuild; all 0 while
 * active domains are off or before t_delay. */
int  crm_debug_activity(crm_t* ctx, uint8_t* flags_by_id);

#ifdef __cplusplus
}
#endif
#endif /* CRM_H */
