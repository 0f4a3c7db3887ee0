/* oracle/crm_oracle.h — TEST INFRASTRUCTURE ONLY (not part of the product).
 *
 * Plain, slow, fp64 CPU oracle of the Chrono::CRM per-step SPH particle update
 * (arXiv 2507.05643; §2.1–§2.5.1 and §4.1).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may
 * load liboracle.so.  It shares no code, header, table or constant generator with
 * paper_2507_05643_b200/ (the CUDA path); neither includes the other.
 *
 * Citation convention: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md
 * line n, "A<k>"/"B<k>" = the readings listed in DESIGN.md §Readings (taken from
 * SURVEY.md §8(c)).
 *
 * Units SI.  Vectors are row-major n×3, stresses n×6 in (xx,yy,zz,xy,xz,yz),
 * tension positive, sigma = -p I + tau.
 */
#ifndef CRM_ORACLE_H
#define CRM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Error codes of the oracle (same meanings as the product's, defined here independently). */
enum {
  OC_OK = 0, OC_E_INVALID = -1, OC_E_DOMAIN = -2, OC_E_NONFINITE = -3,
  OC_E_UNSUPPORTED = -4, OC_E_STATE = -5, OC_E_OOM = -6
};

enum { OC_VISC_BILATERAL = 0, OC_VISC_UNILATERAL = 1 };
enum { OC_BODY_FIXED = 0, OC_BODY_FREE = 1, OC_BODY_PRESCRIBED = 2 };
enum { OC_FLUID = 0, OC_BCE = 1 };

typedef struct {
  /* material, P:296–298 (K, G), P:416–427 (mu_s, mu_2, I0, d, rho0), P:404 (c) */
  double rho0, K, G, mu_s, mu_2, I0, cohesion, grain_d;
  /* SPH discretisation, Table tab:sph_params P:41–58 */
  double d0, h, support;          /* support = kernel support factor (2.0) */
  int    visc_mode;               /* OC_VISC_* (P:361 / P:367) */
  double gamma_a, xi2, cs;        /* xi2 <= 0 -> 0.01 h^2 (A10); cs <= 0 -> sqrt(K/rho0) (A10) */
  double gravity[3];              /* f_b for fluid */
  double lo[3], hi[3];            /* fixed grid box (A19) */
  int    ps_freq;                 /* Alg. 2: lists rebuilt when t mod ps_freq = 0; <= 0 -> 1 */
  int    kernel;                  /* OC_KERNEL_* (quintic Wendland or cubic spline) */
} oc_params;

enum { OC_KERNEL_CUBIC = 0, OC_KERNEL_WENDLAND = 1 };

typedef struct {
  double mass, inertia[3], pos[3], quat[4], vel[3], omega[3];   /* inertia: principal moments about the body axes */
  int motion;                     /* OC_BODY_* */
  int dof_mask;                   /* FREE: bit k set = DOF k free (0..2 translation x,y,z; 3..5 rotation) */
} oc_body;

typedef struct oc_sim oc_sim;

/* ---- pure functions (pinned individually by tests/test_oracle_*.py) ---- */
double oc_W(double r, double h);                      /* cubic spline, A1 */
double oc_dWdr(double r, double h);                   /* dW/dr of the same */
void   oc_gradW(const double xij[3], double h, double out[3]);   /* grad_i W_ij, xij = x_i - x_j */
/* quintic Wendland (Wendland 1995, reading A28), support 2h, and its dW/dr */
double oc_W_wendland(double r, double h);
double oc_dWdr_wendland(double r, double h);
/* paper's linear cell index c = z*(Y*X) + y*X + x */
int64_t oc_paper_cell_index(int64_t x, int64_t y, int64_t z, int64_t X, int64_t Y);
/* B1 binning of one fp32 position; returns OC_E_DOMAIN if outside the grid */
int    oc_cell_coords(const float x[3], const float lo[3], float s, const int dims[3], int out[3]);
/* B2 predicate on fp32 positions: 1 iff |xj - xi| < R (strict) */
int    oc_pair_predicate(const float xi[3], const float xj[3], float R2);
/* O(N^2) all-pairs neighbour sets ("naively by checking all particle pairs") */
int    oc_brute_neighbors(int64_t n, const float* x32, double radius, int64_t* offsets /*n+1*/,
                          int64_t* list /*offsets[n] entries, may be NULL for a count pass*/);
/* Jaumann stress rate d sigma/dt from L (L_ab = d u_a / d x_b) and sigma (A4–A6) */
void   oc_stress_rate(const double L[9], const double sig[6], double K, double G, double out[6]);
/* four-step mu(I) return map (A15–A16); sig_n gives tau_bar^n */
void   oc_return_map(const double sig_star[6], const double sig_n[6], const oc_params* p,
                     double dt, double out[6]);

/* ---- simulation object (same call shape as the product's C-ABI) ---- */
int  oc_create(const oc_params* p, oc_sim** out);
void oc_destroy(oc_sim* s);
int  oc_add_fluid(oc_sim* s, int64_t n, const double* pos, const double* vel, const double* sig6,
                  int64_t* first_id);
int  oc_add_body(oc_sim* s, const oc_body* b, int32_t* body_id);   /* body 0 = static walls */
int  oc_add_bce(oc_sim* s, int32_t body, int64_t n, const double* pos_world, int64_t* first_id);
int  oc_step(oc_sim* s, double dt, int64_t nsteps);
int64_t oc_count(const oc_sim* s, int which /*0 fluid, 1 bce, 2 all*/);
int  oc_get_state(const oc_sim* s, int64_t first, int64_t count, double* pos, double* vel,
                  double* rho, double* sig6);
int  oc_set_state(oc_sim* s, int64_t first, int64_t count, const double* pos, const double* vel,
                  const double* rho, const double* sig6);
int  oc_get_body(const oc_sim* s, int32_t body, oc_body* state, double force[3], double torque[3]);
/* structure of the CURRENT state (what the next oc_step builds first) */
int  oc_structure(oc_sim* s, uint32_t* cell_by_id, int64_t* sorted_ids, uint32_t* nbr_count_by_id,
                  uint32_t* cell_start /* M+1 */, int64_t* n_cells);
/* neighbour sets of the CURRENT state by id: CSR, each row ascending by id */
int  oc_neighbors(oc_sim* s, int64_t* offsets /*n+1*/, int64_t* list /*may be NULL*/);
/* rates of the last step: stage 0 = A (at y_n), 1 = B (at y_mid); fluid rows only meaningful */
int  oc_last_rates(const oc_sim* s, int stage, double* drho, double* acc, double* dsig6);
/* extrapolated BCE velocity/stress of the last step's stage (marker rows only meaningful) */
int  oc_last_bce(const oc_sim* s, int stage, double* vel, double* sig6);

/* ---- active domains (Alg. 3; readings A29–A31) ---- */
enum { OC_ACTIVE = 0, OC_EXTENDED = 1, OC_INACTIVE = 2 };
enum { OC_CAP_KEEP = 0, OC_CAP_GROW = 1, OC_CAP_SHRINK = 2 };
/* UpdateActivity for one point: Active inside the box (body frame, |x_local| <= half), Extended-Active
 * outside every box but closer than `radius` (= 2h) to one, else Inactive (Fig. active_domain).
 * box_pos/box_R/box_half: nbox boxes (3, 9 row-major body->world, 3 doubles each). */
int  oc_activity(const double x[3], int nbox, const double* box_pos, const double* box_R,
                 const double* box_half, double radius);
/* ManageArrayMemory policy: returns the new capacity and the action taken */
int64_t oc_manage_capacity(int64_t capacity, int64_t required, int64_t step, double growth,
                           double shrink, int shrink_interval, int* action);
/* an active box of half extents half[3] at the local origin of `body` (before the first step) */
int  oc_set_active_box(oc_sim* s, int32_t body, const double half[3]);
int  oc_set_active_delay(oc_sim* s, double t_delay);
/* activity flags (by id) of the last list rebuild; all OC_ACTIVE while the feature is off */
int  oc_get_activity(const oc_sim* s, uint8_t* flags);
const char* oc_last_error(const oc_sim* s);
int  oc_num_threads(void);
void oc_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
