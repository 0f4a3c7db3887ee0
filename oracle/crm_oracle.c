/* oracle/crm_oracle.c — TEST INFRASTRUCTURE ONLY (not part of the product).
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of the per-step SPH
 * particle update of Chrono::CRM (arXiv 2507.05643).  It follows the paper's
 * algorithm step by step in the paper's order and notation:
 *
 *   structure  : hash -> sort -> cellStart/cellEnd
 *                -> Alg. 1 neighbour lists with a prefix-sum offset array
 *   stage A    : BCE extrapolation -> rates Eq. continuity_dis /
 *                momentum_dis / stress_rate_dis + artificial viscosity
 *                -> y_mid = y_n + dt/2 f(y_n)
 *   stage B    : the same at y_mid with the SAME neighbour lists (A17)
 *                -> y* = y_n + dt f(y_mid)
 *   return map : Steps 1–4 on sigma*
 *   bodies     : marker accelerations -> force/torque, rigid update (A13)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * It shares no code with paper_2507_05643_b200/.  Gather-only OpenMP loops over
 * particles; built -O2 -fopenmp -ffp-contract=off (no fast-math), so the fp32
 * structural layer (B1–B5) is evaluated with plain IEEE float operations.
 *
 * Parity pins for every function: tests/test_oracle_*.py.
 */
#include "crm_oracle.h"
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OC_MAX_BODIES 64

/* ------------------------------------------------------------------------- */
/* Kernel: cubic spline of Monaghan (1985), support 2h.                       */
/* P:53–55 ("Cubic"), P:726 ("For these kernels in 3D simulations, K = 2");   */
/* coefficients per reading A1: sigma3 = 1/(pi h^3).                          */
/* ------------------------------------------------------------------------- */
double oc_W(double r, double h) {
  const double q = r / h;
  const double sigma3 = 1.0 / (M_PI * h * h * h);
  if (q < 1.0) return sigma3 * (1.0 - 1.5 * q * q + 0.75 * q * q * q);
  if (q < 2.0) {
    const double t = 2.0 - q;
    return sigma3 * 0.25 * t * t * t;
  }
  return 0.0;
}

double oc_dWdr(double r, double h) {
  const double q = r / h;
  const double sigma3 = 1.0 / (M_PI * h * h * h);
  if (q < 1.0) return sigma3 / h * (-3.0 * q + 2.25 * q * q);
  if (q < 2.0) {
    const double t = 2.0 - q;
    return sigma3 / h * (-0.75 * t * t);
  }
  return 0.0;
}

/* grad_i W_ij = dW/dr (r_ij) * (x_i - x_j)/r_ij; zero at r = 0 (A18). */
void oc_gradW(const double xij[3], double h, double out[3]) {
  const double r = sqrt(xij[0] * xij[0] + xij[1] * xij[1] + xij[2] * xij[2]);
  if (r == 0.0) { out[0] = out[1] = out[2] = 0.0; return; }
  const double f = oc_dWdr(r, h) / r;
  out[0] = f * xij[0]; out[1] = f * xij[1]; out[2] = f * xij[2];
}

/* ------------------------------------------------------------------------- */
/* Kernel: quintic Wendland (Wendland 1995), support 2h (reading A28):  */
/* the degree-5 compactly supported function W = a (1 - q/2)^4 (2q + 1),      */
/* a = 21 / (16 pi h^3) in 3D, q = r/h <= 2.                                   */
/* ------------------------------------------------------------------------- */
double oc_W_wendland(double r, double h) {
  const double q = r / h;
  if (q >= 2.0) return 0.0;
  const double a = 21.0 / (16.0 * M_PI * h * h * h);
  const double t = 1.0 - 0.5 * q;
  return a * t * t * t * t * (2.0 * q + 1.0);
}

/* d/dr of the above: a/h * [-2 t^3 (2q + 1) + 2 t^4] = -5 a q t^3 / h */
double oc_dWdr_wendland(double r, double h) {
  const double q = r / h;
  if (q >= 2.0) return 0.0;
  const double a = 21.0 / (16.0 * M_PI * h * h * h);
  const double t = 1.0 - 0.5 * q;
  return -5.0 * a * q * t * t * t / h;
}

/* the kernel the simulation uses (oc_params.kernel) */
static double sim_W(const oc_params* p, double r) {
  return p->kernel == OC_KERNEL_WENDLAND ? oc_W_wendland(r, p->h) : oc_W(r, p->h);
}

static void sim_gradW(const oc_params* p, const double xij[3], double out[3]) {
  if (p->kernel != OC_KERNEL_WENDLAND) { oc_gradW(xij, p->h, out); return; }
  const double r = sqrt(xij[0] * xij[0] + xij[1] * xij[1] + xij[2] * xij[2]);
  if (r == 0.0) { out[0] = out[1] = out[2] = 0.0; return; }
  const double f = oc_dWdr_wendland(r, p->h) / r;
  out[0] = f * xij[0]; out[1] = f * xij[1]; out[2] = f * xij[2];
}

/* ------------------------------------------------------------------------- */
/* Structural layer (Alg. 1) on fp32 positions, rules B1–B5.        */
/* ------------------------------------------------------------------------- */
/* c = z * (Y_size * X_size) + y * X_size + x. */
int64_t oc_paper_cell_index(int64_t x, int64_t y, int64_t z, int64_t X, int64_t Y) {
  return z * (Y * X) + y * X + x;
}

/* B1: c_a = floor((x_a - o_a) / s) in IEEE fp32, round-to-nearest division. */
int oc_cell_coords(const float x[3], const float lo[3], float s, const int dims[3], int out[3]) {
  for (int a = 0; a < 3; ++a) {
    const float t = (x[a] - lo[a]) / s;
    const float f = floorf(t);
    if (!(f >= 0.0f) || f >= (float)dims[a]) return OC_E_DOMAIN;   /* also catches NaN */
    out[a] = (int)f;
  }
  return OC_OK;
}

/* B2: dx = xj - xi; r2 = fma(dz,dz, fma(dy,dy, dx*dx)); neighbour iff r2 < R2 (P:758 strict). */
int oc_pair_predicate(const float xi[3], const float xj[3], float R2) {
  const float dx = xj[0] - xi[0];
  const float dy = xj[1] - xi[1];
  const float dz = xj[2] - xi[2];
  const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
  return r2 < R2;
}

/* O(N^2) definition of the neighbour set {(i,j): i != j, |x_i - x_j| < 2h}. */
int oc_brute_neighbors(int64_t n, const float* x32, double radius, int64_t* offsets, int64_t* list) {
  const float R2 = (float)(radius * radius);
  offsets[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      if (oc_pair_predicate(&x32[3 * i], &x32[3 * j], R2)) {
        if (list) list[offsets[i] + c] = j;
        ++c;
      }
    }
    offsets[i + 1] = offsets[i] + c;
  }
  return OC_OK;
}

/* ------------------------------------------------------------------------- */
/* Constitutive pieces                                                        */
/* ------------------------------------------------------------------------- */
/* symmetric 6-vector (xx,yy,zz,xy,xz,yz) <-> 3x3 */
static void sym_to_mat(const double s[6], double m[9]) {
  m[0] = s[0]; m[1] = s[3]; m[2] = s[4];
  m[3] = s[3]; m[4] = s[1]; m[5] = s[5];
  m[6] = s[4]; m[7] = s[5]; m[8] = s[2];
}

/* Eq. equ:stress_rate with Eq. 3:
 *   d sigma/dt = phi_dot sigma - sigma phi_dot + 2G (eps_dot - 1/3 tr(eps_dot) I) + K tr(eps_dot) I
 * eps_dot = 1/2 (L + L^T) (elastic part only), phi_dot = 1/2 (L - L^T),
 * L_ab = d u_a / d x_b (A4, A5); bulk coefficient K per Eq. 3 (A6). */
void oc_stress_rate(const double L[9], const double sig[6], double K, double G, double out[6]) {
  double S[9], E[9], Om[9], R[9];
  sym_to_mat(sig, S);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      E[3 * a + b] = 0.5 * (L[3 * a + b] + L[3 * b + a]);
      Om[3 * a + b] = 0.5 * (L[3 * a + b] - L[3 * b + a]);
    }
  const double tr = E[0] + E[4] + E[8];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double os = 0.0, so = 0.0;
      for (int k = 0; k < 3; ++k) {
        os += Om[3 * a + k] * S[3 * k + b];
        so += S[3 * a + k] * Om[3 * k + b];
      }
      const double d = (a == b) ? 1.0 : 0.0;
      R[3 * a + b] = os - so + 2.0 * G * (E[3 * a + b] - tr / 3.0 * d) + K * tr * d;
    }
  out[0] = R[0]; out[1] = R[4]; out[2] = R[8];
  out[3] = R[1]; out[4] = R[2]; out[5] = R[5];
}

/* Eq. eq:trial_quantities: p = -tr(s)/3, tau = s + p I, tau_bar = sqrt(1/2 tau:tau) */
static void trial_quantities(const double s[6], double* p, double tau[6], double* tau_bar) {
  *p = -(s[0] + s[1] + s[2]) / 3.0;
  tau[0] = s[0] + *p; tau[1] = s[1] + *p; tau[2] = s[2] + *p;
  tau[3] = s[3]; tau[4] = s[4]; tau[5] = s[5];
  const double tt = tau[0] * tau[0] + tau[1] * tau[1] + tau[2] * tau[2]
                  + 2.0 * (tau[3] * tau[3] + tau[4] * tau[4] + tau[5] * tau[5]);
  *tau_bar = sqrt(0.5 * tt);
}

/* Return mapping, Steps 1–4; readings A15 (after the full step only),
 * A16 (gamma_dot >= 0, p floored at 1 Pa for I only, I = 0 -> mu = mu_s,
 * tau_bar^n recomputed from sigma_n), A27 (tau_max floored at 0). */
void oc_return_map(const double sig_star[6], const double sig_n[6], const oc_params* P,
                   double dt, double out[6]) {
  double p_star, tau_star[6], tb_star;
  trial_quantities(sig_star, &p_star, tau_star, &tb_star);
  /* Step 1: tension cut-off, Eq. eq:pcrit */
  const double p_cri = -P->cohesion / P->mu_s;
  if (p_star < p_cri) { for (int k = 0; k < 6; ++k) out[k] = 0.0; return; }
  /* Step 2: mu(I) rheology, Eq. eq:muI */
  double p_n, tau_n[6], tb_n;
  trial_quantities(sig_n, &p_n, tau_n, &tb_n);
  double gamma_dot = (tb_star - tb_n) / (P->G * dt);
  if (gamma_dot < 0.0) gamma_dot = 0.0;
  const double p_for_I = p_star > 1.0 ? p_star : 1.0;
  const double I = gamma_dot * P->grain_d * sqrt(P->rho0 / p_for_I);
  const double mu = (I > 0.0) ? P->mu_s + (P->mu_2 - P->mu_s) / (1.0 + P->I0 / I) : P->mu_s;
  /* Step 3: yield test, Eq. eq:yieldsurf */
  double tau_max = mu * p_star + P->cohesion;
  if (tau_max < 0.0) tau_max = 0.0;
  if (tb_star <= tau_max) { for (int k = 0; k < 6; ++k) out[k] = sig_star[k]; return; }
  /* Step 4: radial return */
  const double scale = tau_max / tb_star;
  for (int k = 0; k < 6; ++k) out[k] = scale * tau_star[k];
  out[0] -= p_star; out[1] -= p_star; out[2] -= p_star;
}

/* ------------------------------------------------------------------------- */
/* Simulation object                                                          */
/* ------------------------------------------------------------------------- */
typedef struct {
  oc_body b;
  double acc[3], alpha[3];   /* last rigid accelerations (used in BCE stress extrapolation) */
  double force[3], torque[3];
} body_rec;

struct oc_sim {
  oc_params P;
  double m;                   /* particle mass rho0 d0^3 */
  double xi2, cs, R;          /* resolved xi^2, c_s, support radius support*h */
  int64_t n, cap, n_fluid, n_bce;
  int* kind; int* body;
  double *x, *u, *rho, *sig;  /* by id */
  double* xl;                 /* marker position in its body's frame */
  int nb; body_rec bodies[OC_MAX_BODIES];
  int64_t steps_done;
  double time;                /* t = sum of the step sizes taken (Alg. 3 compares it with t_delay) */
  void* kept;                 /* structure_t of the last rebuild (Alg. 2) */
  int has_box[OC_MAX_BODIES]; /* active boxes (Alg. 3): half extents at each body's local origin */
  double box_half[OC_MAX_BODIES][3];
  double t_delay;
  double* rates[2];           /* per stage: n * 10 (drho, acc3, dsig6) */
  double* bce[2];             /* per stage: n * 9 (u3, sig6) */
  char err[256];
};

static int grow(oc_sim* s, int64_t need) {
  if (need <= s->cap) return OC_OK;
  int64_t nc = s->cap ? s->cap : 1024;
  while (nc < need) nc *= 2;
#define RE(p, k) do { void* t = realloc(p, (size_t)nc * (k) * sizeof(*(p))); if (!t) return OC_E_OOM; p = t; } while (0)
  RE(s->kind, 1); RE(s->body, 1); RE(s->x, 3); RE(s->u, 3); RE(s->rho, 1); RE(s->sig, 6); RE(s->xl, 3);
  RE(s->rates[0], 10); RE(s->rates[1], 10); RE(s->bce[0], 9); RE(s->bce[1], 9);
#undef RE
  s->cap = nc;
  return OC_OK;
}

int oc_create(const oc_params* p, oc_sim** out) {
  *out = NULL;
  if (!p) return OC_E_INVALID;
  /* S:31, S:35, S:91 parameter validity */
  if (!(p->h > 0) || !(p->d0 > 0) || p->h < p->d0 || !(p->rho0 > 0) || !(p->K > 0) || !(p->G > 0)
      || !(p->mu_s > 0) || p->mu_s > p->mu_2 || !(p->I0 > 0) || p->cohesion < 0 || !(p->grain_d > 0)
      || p->gamma_a < 0)
    return OC_E_INVALID;
  if (p->support != 0.0 && p->support != 2.0) return OC_E_UNSUPPORTED;  /* both kernels: support 2h */
  if (p->kernel != OC_KERNEL_CUBIC && p->kernel != OC_KERNEL_WENDLAND) return OC_E_INVALID;
  for (int a = 0; a < 3; ++a) if (!(p->hi[a] > p->lo[a])) return OC_E_INVALID;
  oc_sim* s = (oc_sim*)calloc(1, sizeof(oc_sim));
  if (!s) return OC_E_OOM;
  s->P = *p;
  if (s->P.support == 0.0) s->P.support = 2.0;
  s->m = p->rho0 * p->d0 * p->d0 * p->d0;
  s->xi2 = p->xi2 > 0 ? p->xi2 : 0.01 * p->h * p->h;
  s->cs = p->cs > 0 ? p->cs : sqrt(p->K / p->rho0);
  s->R = s->P.support * p->h;
  /* body 0: the static walls (identity pose) */
  s->nb = 1;
  memset(&s->bodies[0], 0, sizeof(body_rec));
  s->bodies[0].b.quat[0] = 1.0;
  s->bodies[0].b.motion = OC_BODY_FIXED;
  *out = s;
  return OC_OK;
}

static void drop_kept(oc_sim* s);
static uint8_t* compute_activity(const oc_sim* s);

void oc_destroy(oc_sim* s) {
  if (!s) return;
  free(s->kind); free(s->body); free(s->x); free(s->u); free(s->rho); free(s->sig); free(s->xl);
  free(s->rates[0]); free(s->rates[1]); free(s->bce[0]); free(s->bce[1]);
  drop_kept(s);
  free(s);
}

int oc_add_fluid(oc_sim* s, int64_t n, const double* pos, const double* vel, const double* sig6,
                 int64_t* first_id) {
  if (s->steps_done > 0) return OC_E_STATE;
  if (n < 0 || (n > 0 && !pos)) return OC_E_INVALID;
  int r = grow(s, s->n + n); if (r) return r;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = s->n + k;
    s->kind[i] = OC_FLUID; s->body[i] = -1;
    for (int a = 0; a < 3; ++a) { s->x[3 * i + a] = pos[3 * k + a]; s->u[3 * i + a] = vel ? vel[3 * k + a] : 0.0; s->xl[3 * i + a] = 0; }
    s->rho[i] = s->P.rho0;
    for (int c = 0; c < 6; ++c) s->sig[6 * i + c] = sig6 ? sig6[6 * k + c] : 0.0;
  }
  if (first_id) *first_id = s->n;
  s->n += n; s->n_fluid += n;
  return OC_OK;
}

/* quaternion (w,x,y,z) -> rotation matrix */
static void quat_to_R(const double q[4], double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

/* q <- exp(tau * omega / 2) (x) q  (rotation by |omega| tau about omega) */
static void quat_advance(double q[4], const double w[3], double tau) {
  const double wn = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  if (wn == 0.0) return;
  const double ang = 0.5 * wn * tau, c = cos(ang), sn = sin(ang) / wn;
  const double d[4] = {c, sn * w[0], sn * w[1], sn * w[2]};
  const double r[4] = {
    d[0] * q[0] - d[1] * q[1] - d[2] * q[2] - d[3] * q[3],
    d[0] * q[1] + d[1] * q[0] + d[2] * q[3] - d[3] * q[2],
    d[0] * q[2] - d[1] * q[3] + d[2] * q[0] + d[3] * q[1],
    d[0] * q[3] + d[1] * q[2] - d[2] * q[1] + d[3] * q[0]};
  const double nn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2] + r[3] * r[3]);
  for (int k = 0; k < 4; ++k) q[k] = r[k] / nn;
}

int oc_add_body(oc_sim* s, const oc_body* b, int32_t* body_id) {
  if (s->steps_done > 0) return OC_E_STATE;
  if (!b || s->nb >= OC_MAX_BODIES) return OC_E_INVALID;
  if (b->motion == OC_BODY_FREE && !(b->mass > 0)) return OC_E_INVALID;
  body_rec* r = &s->bodies[s->nb];
  memset(r, 0, sizeof(*r));
  r->b = *b;
  const double qn = sqrt(b->quat[0] * b->quat[0] + b->quat[1] * b->quat[1] + b->quat[2] * b->quat[2] + b->quat[3] * b->quat[3]);
  if (!(qn > 0)) return OC_E_INVALID;
  for (int k = 0; k < 4; ++k) r->b.quat[k] = b->quat[k] / qn;
  if (body_id) *body_id = s->nb;
  s->nb++;
  return OC_OK;
}

int oc_add_bce(oc_sim* s, int32_t body, int64_t n, const double* pos_world, int64_t* first_id) {
  if (s->steps_done > 0) return OC_E_STATE;
  if (body < 0 || body >= s->nb || n < 0 || (n > 0 && !pos_world)) return OC_E_INVALID;
  int r = grow(s, s->n + n); if (r) return r;
  const oc_body* b = &s->bodies[body].b;
  double R[9]; quat_to_R(b->quat, R);
  for (int64_t k = 0; k < n; ++k) {
    const int64_t i = s->n + k;
    s->kind[i] = OC_BCE; s->body[i] = body;
    double d[3];
    for (int a = 0; a < 3; ++a) { s->x[3 * i + a] = pos_world[3 * k + a]; d[a] = pos_world[3 * k + a] - b->pos[a]; s->u[3 * i + a] = 0.0; }
    for (int a = 0; a < 3; ++a) s->xl[3 * i + a] = R[0 + a] * d[0] + R[3 + a] * d[1] + R[6 + a] * d[2];  /* R^T d */
    s->rho[i] = s->P.rho0;     /* A8: rho_a = rho0 */
    for (int c = 0; c < 6; ++c) s->sig[6 * i + c] = 0.0;
  }
  if (first_id) *first_id = s->n;
  s->n += n; s->n_bce += n;
  return OC_OK;
}

int64_t oc_count(const oc_sim* s, int which) {
  return which == 0 ? s->n_fluid : which == 1 ? s->n_bce : s->n;
}

/* ---- structure: hash, sort, cellStart, Alg. 1 ---------------------------- */
typedef struct {
  int dims[3]; int64_t M;
  uint32_t* cell;        /* by id */
  int64_t* sorted;       /* sorted index -> id */
  uint32_t* cell_start;  /* M+1 */
  int64_t* offset;       /* by id, n+1 (CSR of neighbour ids) */
  int64_t* list;
  uint8_t* act;          /* by id: OC_ACTIVE / OC_EXTENDED / OC_INACTIVE; NULL = all active (Alg. 3 off) */
} structure_t;

static void free_structure(structure_t* st) {
  free(st->cell); free(st->sorted); free(st->cell_start); free(st->offset); free(st->list); free(st->act);
  memset(st, 0, sizeof(*st));
}

static void drop_kept(oc_sim* s) {
  if (!s->kept) return;
  free_structure((structure_t*)s->kept);
  free(s->kept);
  s->kept = NULL;
}

static const uint32_t* g_sort_cell;   /* qsort context (single-threaded) */
static int cmp_cell_id(const void* a, const void* b) {
  const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
  const uint32_t ca = g_sort_cell[ia], cb = g_sort_cell[ib];
  if (ca != cb) return ca < cb ? -1 : 1;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* act (by id, may be NULL) is owned by st afterwards: Inactive particles (Alg. 3) take no part in
 * the structure: no cell (sentinel M), sorted behind every active particle, no neighbours, nobody's
 * neighbour ("they are not included in neighbor search"). */
static int build_structure(oc_sim* s, const double* x, structure_t* st, int want_list, uint8_t* act) {
  memset(st, 0, sizeof(*st));
  st->act = act;
  const int64_t n = s->n;
  const double sd = s->R;                    /* cell size = 2h */
  const float s32 = (float)sd;
  float lo32[3];
  for (int a = 0; a < 3; ++a) {
    lo32[a] = (float)s->P.lo[a];
    st->dims[a] = (int)ceil((s->P.hi[a] - s->P.lo[a]) / sd);
  }
  /* axes relabelled for the paper's formula: paper x := our z (fastest), paper z := our x (B3) */
  const int X = st->dims[2], Y = st->dims[1];
  st->M = (int64_t)st->dims[0] * st->dims[1] * st->dims[2];
  float* x32 = (float*)malloc((size_t)(n ? n : 1) * 3 * sizeof(float));
  st->cell = (uint32_t*)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
  st->sorted = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  st->cell_start = (uint32_t*)calloc((size_t)st->M + 1, sizeof(uint32_t));
  if (!x32 || !st->cell || !st->sorted || !st->cell_start) { free(x32); free_structure(st); return OC_E_OOM; }
  for (int64_t i = 0; i < 3 * n; ++i) x32[i] = (float)x[i];
  /* Step 1: hash every particle */
  for (int64_t i = 0; i < n; ++i) {
    int c[3];
    if (act && act[i] == OC_INACTIVE) { st->cell[i] = (uint32_t)st->M; continue; }
    if (oc_cell_coords(&x32[3 * i], lo32, s32, st->dims, c) != OC_OK) {
      snprintf(s->err, sizeof s->err, "particle id %lld outside the grid at step %lld",
               (long long)i, (long long)s->steps_done);
      free(x32); free_structure(st); return OC_E_DOMAIN;
    }
    st->cell[i] = (uint32_t)oc_paper_cell_index(c[2], c[1], c[0], X, Y);
  }
  /* Step 2: sort by (cell, id) (B4) */
  for (int64_t i = 0; i < n; ++i) st->sorted[i] = i;
  g_sort_cell = st->cell;
  qsort(st->sorted, (size_t)n, sizeof(int64_t), cmp_cell_id);
  /* Step 3: cellStart / cellEnd; cellEnd[c] = cellStart[c+1] (CSR, B4) */
  for (int64_t i = 0; i < n; ++i)
    if (st->cell[i] < (uint32_t)st->M) st->cell_start[st->cell[i] + 1]++;
  for (int64_t c = 0; c < st->M; ++c) st->cell_start[c + 1] += st->cell_start[c];
  if (!want_list) { free(x32); return OC_OK; }
  /* Step 4 (Alg. 1): per sorted particle, 27 cells, strict < 2h.
   * The offset array is the prefix sum of a counting pass identical in traversal. */
  const float R2 = (float)(sd * sd);
  int64_t* cnt = (int64_t*)calloc((size_t)(n ? n : 1), sizeof(int64_t));
  st->offset = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  if (!cnt || !st->offset) { free(cnt); free(x32); free_structure(st); return OC_E_OOM; }
  for (int pass = 0; pass < 2; ++pass) {
    #pragma omp parallel for schedule(dynamic, 256)
    for (int64_t si = 0; si < n; ++si) {
      const int64_t i = st->sorted[si];
      int64_t count = 0;
      if (st->cell[i] >= (uint32_t)st->M) { if (pass == 0) cnt[i] = 0; continue; }   /* Inactive */
      int g[3];
      oc_cell_coords(&x32[3 * i], lo32, s32, st->dims, g);      /* calcGridPos */
      for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dz = -1; dz <= 1; ++dz) {
            const int nx = g[0] + dx, ny = g[1] + dy, nz = g[2] + dz;
            if (nx < 0 || ny < 0 || nz < 0 || nx >= st->dims[0] || ny >= st->dims[1] || nz >= st->dims[2]) continue;
            const int64_t gid = oc_paper_cell_index(nz, ny, nx, X, Y);   /* calcGridID */
            for (uint32_t sj = st->cell_start[gid]; sj < st->cell_start[gid + 1]; ++sj) {
              const int64_t j = st->sorted[sj];
              if (j == i) continue;                                      /* A18 */
              if (oc_pair_predicate(&x32[3 * i], &x32[3 * j], R2)) {
                if (pass == 1) st->list[st->offset[i] + count] = j;
                ++count;
              }
            }
          }
      if (pass == 0) cnt[i] = count;
    }
    if (pass == 0) {
      for (int64_t i = 0; i < n; ++i) st->offset[i + 1] = st->offset[i] + cnt[i];
      st->list = (int64_t*)malloc((size_t)(st->offset[n] ? st->offset[n] : 1) * sizeof(int64_t));
      if (!st->list) { free(cnt); free(x32); free_structure(st); return OC_E_OOM; }
    }
  }
  free(cnt); free(x32);
  return OC_OK;
}

int oc_structure(oc_sim* s, uint32_t* cell_by_id, int64_t* sorted_ids, uint32_t* nbr_count_by_id,
                 uint32_t* cell_start, int64_t* n_cells) {
  structure_t st;
  int r = build_structure(s, s->x, &st, nbr_count_by_id != NULL, compute_activity(s));
  if (r) return r;
  if (cell_by_id) memcpy(cell_by_id, st.cell, (size_t)s->n * sizeof(uint32_t));
  if (sorted_ids) memcpy(sorted_ids, st.sorted, (size_t)s->n * sizeof(int64_t));
  if (nbr_count_by_id)
    for (int64_t i = 0; i < s->n; ++i) nbr_count_by_id[i] = (uint32_t)(st.offset[i + 1] - st.offset[i]);
  if (cell_start) memcpy(cell_start, st.cell_start, (size_t)(st.M + 1) * sizeof(uint32_t));
  if (n_cells) *n_cells = st.M;
  free_structure(&st);
  return OC_OK;
}

int oc_neighbors(oc_sim* s, int64_t* offsets, int64_t* list) {
  structure_t st;
  int r = build_structure(s, s->x, &st, 1, compute_activity(s));
  if (r) return r;
  memcpy(offsets, st.offset, (size_t)(s->n + 1) * sizeof(int64_t));
  if (list) {
    memcpy(list, st.list, (size_t)st.offset[s->n] * sizeof(int64_t));
    for (int64_t i = 0; i < s->n; ++i)
      qsort(list + offsets[i], (size_t)(offsets[i + 1] - offsets[i]), sizeof(int64_t), cmp_i64);
  }
  free_structure(&st);
  return OC_OK;
}

/* ---- bodies: marker kinematics ------------------------------------------- */
typedef struct { double pos[3], R[9], vel[3], omega[3], acc[3], alpha[3]; } pose_t;

static void body_pose(const body_rec* r, double tau, pose_t* out) {
  /* pose advanced kinematically by tau with the current velocities (prescribed and free
   * bodies keep their velocity within a step; the rigid update happens once per step) */
  double q[4] = {r->b.quat[0], r->b.quat[1], r->b.quat[2], r->b.quat[3]};
  for (int a = 0; a < 3; ++a) {
    out->pos[a] = r->b.pos[a] + tau * r->b.vel[a];
    out->vel[a] = r->b.vel[a]; out->omega[a] = r->b.omega[a];
    out->acc[a] = r->acc[a]; out->alpha[a] = r->alpha[a];
  }
  quat_advance(q, r->b.omega, tau);
  quat_to_R(q, out->R);
}

static void cross(const double a[3], const double b[3], double c[3]) {
  c[0] = a[1] * b[2] - a[2] * b[1];
  c[1] = a[2] * b[0] - a[0] * b[2];
  c[2] = a[0] * b[1] - a[1] * b[0];
}

/* marker world position, body velocity and body acceleration at the marker */
static void marker_kinematics(const oc_sim* s, const pose_t* poses, int64_t i,
                              double xw[3], double ub[3], double ab[3]) {
  const int b = s->body[i];
  const pose_t* P = &poses[b];
  const double* xl = &s->xl[3 * i];
  double r[3];
  for (int a = 0; a < 3; ++a) r[a] = P->R[3 * a] * xl[0] + P->R[3 * a + 1] * xl[1] + P->R[3 * a + 2] * xl[2];
  for (int a = 0; a < 3; ++a) xw[a] = P->pos[a] + r[a];
  double wr[3], wwr[3], ar[3];
  cross(P->omega, r, wr); cross(P->omega, wr, wwr); cross(P->alpha, r, ar);
  for (int a = 0; a < 3; ++a) { ub[a] = P->vel[a] + wr[a]; ab[a] = P->acc[a] + ar[a] + wwr[a]; }
}

/* ---- active domains (Alg. 3) ----------------------------------- */
/* UpdateActivity: "Particles residing within an active box are flagged as Active ...
 * particles outside an active box but within a distance 2h of its boundary are flagged as
 * Extended-Active ... All remaining particles are flagged as Inactive."  The box is an OOBB at the
 * body's local origin; the distance to it is the Euclidean distance to the solid box
 * (reading A29), evaluated in fp64 (rule B6). */
int oc_activity(const double x[3], int nbox, const double* box_pos, const double* box_R,
                const double* box_half, double radius) {
  int ext = 0;
  for (int b = 0; b < nbox; ++b) {
    const double* p = &box_pos[3 * b];
    const double* R = &box_R[9 * b];
    const double* hb = &box_half[3 * b];
    const double d[3] = {x[0] - p[0], x[1] - p[1], x[2] - p[2]};
    double dist2 = 0.0;
    int inside = 1;
    for (int a = 0; a < 3; ++a) {
      const double l = R[a] * d[0] + R[3 + a] * d[1] + R[6 + a] * d[2];   /* body frame: R^T d */
      const double o = fabs(l) - hb[a];
      if (o > 0.0) { inside = 0; dist2 += o * o; }
    }
    if (inside) return OC_ACTIVE;
    if (dist2 < radius * radius) ext = 1;
  }
  return ext ? OC_EXTENDED : OC_INACTIVE;
}

/* ManageArrayMemory: grow to N_{a+e} G when N_{a+e} exceeds the capacity; every S_I steps,
 * shrink to N_{a+e} when N_{a+e} / capacity < S; otherwise keep. */
int64_t oc_manage_capacity(int64_t capacity, int64_t required, int64_t step, double growth,
                           double shrink, int shrink_interval, int* action) {
  int act = OC_CAP_KEEP;
  int64_t cap = capacity;
  if (required > capacity) {
    act = OC_CAP_GROW;
    cap = (int64_t)ceil((double)required * growth);
  } else if (shrink_interval > 0 && step % shrink_interval == 0 && capacity > 0 &&
             (double)required / (double)capacity < shrink) {
    act = OC_CAP_SHRINK;
    cap = required;
  }
  if (action) *action = act;
  return cap;
}

int oc_set_active_box(oc_sim* s, int32_t body, const double half[3]) {
  if (s->steps_done > 0) return OC_E_STATE;
  if (body < 0 || body >= s->nb || !half) return OC_E_INVALID;
  for (int a = 0; a < 3; ++a) if (!(half[a] >= 0.0)) return OC_E_INVALID;
  s->has_box[body] = 1;
  for (int a = 0; a < 3; ++a) s->box_half[body][a] = half[a];
  drop_kept(s);
  return OC_OK;
}

int oc_set_active_delay(oc_sim* s, double t_delay) {
  s->t_delay = t_delay;
  drop_kept(s);
  return OC_OK;
}

/* flags of every particle at the current state and time, or NULL while Alg. 3 is off
 * ("if t > t_delay", Alg. 3); markers of moving bodies are always Active (reading A29) */
static uint8_t* compute_activity(const oc_sim* s) {
  int nbox = 0;
  double bp[3 * OC_MAX_BODIES], bR[9 * OC_MAX_BODIES], bh[3 * OC_MAX_BODIES];
  for (int b = 0; b < s->nb; ++b) {
    if (!s->has_box[b]) continue;
    pose_t P;
    body_pose(&s->bodies[b], 0.0, &P);
    for (int a = 0; a < 3; ++a) { bp[3 * nbox + a] = P.pos[a]; bh[3 * nbox + a] = s->box_half[b][a]; }
    for (int k = 0; k < 9; ++k) bR[9 * nbox + k] = P.R[k];
    ++nbox;
  }
  if (nbox == 0 || !(s->time > s->t_delay)) return NULL;
  uint8_t* act = (uint8_t*)malloc((size_t)(s->n ? s->n : 1));
  if (!act) return NULL;
  for (int64_t i = 0; i < s->n; ++i) {
    const int moving_marker = s->kind[i] == OC_BCE && s->bodies[s->body[i]].b.motion != OC_BODY_FIXED;
    act[i] = moving_marker ? OC_ACTIVE : (uint8_t)oc_activity(&s->x[3 * i], nbox, bp, bR, bh, s->R);
  }
  return act;
}

int oc_get_activity(const oc_sim* s, uint8_t* flags) {
  const structure_t* st = (const structure_t*)s->kept;
  for (int64_t i = 0; i < s->n; ++i) flags[i] = (st && st->act) ? st->act[i] : OC_ACTIVE;
  return OC_OK;
}

/* Alg. 3, reading A31: only Active particles are updated.  "SPH particles outside active boxes are
 * deactivated ... their states are not updated"; the Extended-Active ones (outside the box,
 * within 2h of it) are kept "to ensure their data is available for these calculations":
 * they are neighbours of Active particles, but their own state (fluid y; marker u, sigma) is frozen. */
static int frozen(const structure_t* st, int64_t i) { return st->act && st->act[i] != OC_ACTIVE; }

/* ---- BCE extrapolation, Adami + stress (reading A12) ---- */
static void bce_extrapolate(const oc_sim* s, const structure_t* st, const double* x, const double* u,
                            const double* rho, const double* sig, const double* ubody,
                            const double* abody, double* u_out, double* sig_out) {
  const double h = s->P.h;
  const double* g = s->P.gravity;
  #pragma omp parallel for schedule(dynamic, 256)
  for (int64_t a = 0; a < s->n; ++a) {
    if (s->kind[a] != OC_BCE) continue;
    if (frozen(st, a)) {   /* Alg. 3: "their states are not updated", A31 */
      for (int c = 0; c < 3; ++c) u_out[3 * a + c] = u[3 * a + c];
      for (int c = 0; c < 6; ++c) sig_out[6 * a + c] = sig[6 * a + c];
      continue;
    }
    double SW = 0.0, su[3] = {0, 0, 0}, ss[6] = {0, 0, 0, 0, 0, 0}, sh = 0.0;
    for (int64_t k = st->offset[a]; k < st->offset[a + 1]; ++k) {
      const int64_t f = st->list[k];
      if (s->kind[f] != OC_FLUID) continue;                 /* b: nearby fluid SPH particles */
      double xaf[3];
      for (int c = 0; c < 3; ++c) xaf[c] = x[3 * a + c] - x[3 * f + c];
      const double W = sim_W(&s->P, sqrt(xaf[0] * xaf[0] + xaf[1] * xaf[1] + xaf[2] * xaf[2]));
      SW += W;
      for (int c = 0; c < 3; ++c) su[c] += u[3 * f + c] * W;
      for (int c = 0; c < 6; ++c) ss[c] += sig[6 * f + c] * W;
      double gd = 0.0;
      for (int c = 0; c < 3; ++c) gd += (g[c] - abody[3 * a + c]) * xaf[c];
      sh += rho[f] * gd * W;
    }
    if (SW > 0.0) {
      /* u_tilde = sum u_b W / sum W; no-slip u_a = 2 u_body - u_tilde */
      for (int c = 0; c < 3; ++c) u_out[3 * a + c] = 2.0 * ubody[3 * a + c] - su[c] / SW;
      for (int c = 0; c < 6; ++c) sig_out[6 * a + c] = ss[c] / SW;
      for (int c = 0; c < 3; ++c) sig_out[6 * a + c] -= sh / SW;
    } else {   /* A11: no fluid neighbour */
      for (int c = 0; c < 3; ++c) u_out[3 * a + c] = ubody[3 * a + c];
      for (int c = 0; c < 6; ++c) sig_out[6 * a + c] = 0.0;
    }
  }
}

/* (sigma . g)_a for symmetric sigma in 6-vector form */
static void sym_dot(const double s[6], const double g[3], double out[3]) {
  out[0] = s[0] * g[0] + s[3] * g[1] + s[4] * g[2];
  out[1] = s[3] * g[0] + s[1] * g[1] + s[5] * g[2];
  out[2] = s[4] * g[0] + s[5] * g[1] + s[2] * g[2];
}

/* ---- SPH rates, Eqs. continuity_dis, momentum_dis, stress_rate_dis, AV ---- */
/* For fluid i: sums over P(i) (fluid and BCE neighbours, A8), kernel at the current
 * positions with W = grad W = 0 for r >= 2h (A17).  For markers of moving bodies: the
 * momentum equation over fluid neighbours only, no gravity (A13). */
static void rates(const oc_sim* s, const structure_t* st, const double* x, const double* u,
                  const double* rho, const double* sig, double* out /* n*10 */) {
  const double h = s->P.h, m = s->m, R = s->R;
  const double av = s->P.gamma_a * h * s->cs;      /* gamma_a h c_s */
  #pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < s->n; ++i) {
    double* o = &out[10 * i];
    for (int c = 0; c < 10; ++c) o[c] = 0.0;
    const int is_fluid = s->kind[i] == OC_FLUID;
    if (!is_fluid && (s->body[i] <= 0 || s->bodies[s->body[i]].b.motion == OC_BODY_FIXED)) continue;
    if (frozen(st, i)) continue;                                      /* Alg. 3, A31: no RHS */
    double L[9] = {0}, cont = 0.0, mom[3] = {0, 0, 0}, Pi[3] = {0, 0, 0};
    for (int64_t k = st->offset[i]; k < st->offset[i + 1]; ++k) {
      const int64_t j = st->list[k];
      if (!is_fluid && s->kind[j] != OC_FLUID) continue;
      double xij[3];
      for (int c = 0; c < 3; ++c) xij[c] = x[3 * i + c] - x[3 * j + c];
      const double r2 = xij[0] * xij[0] + xij[1] * xij[1] + xij[2] * xij[2];
      if (sqrt(r2) >= R) continue;
      double gW[3];
      sim_gradW(&s->P, xij, gW);
      const double Vj = m / rho[j];                                   /* A7 */
      double uji[3];
      for (int c = 0; c < 3; ++c) uji[c] = u[3 * j + c] - u[3 * i + c];
      /* Eq. continuity_dis: -rho_i sum (u_j - u_i) . grad_i W_ij V_j */
      cont += (uji[0] * gW[0] + uji[1] * gW[1] + uji[2] * gW[2]) * Vj;
      /* velocity gradient L = sum V_j u_ji (x) grad_i W_ij (F2, A4) */
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) L[3 * a + b] += Vj * uji[a] * gW[b];
      /* Eq. momentum_dis: (sigma_j + sigma_i) . grad_i W_ij V_j (F3) */
      double ssum[6], sg[3];
      for (int c = 0; c < 6; ++c) ssum[c] = sig[6 * j + c] + sig[6 * i + c];
      sym_dot(ssum, gW, sg);
      for (int c = 0; c < 3; ++c) mom[c] += sg[c] * Vj;
      /* artificial viscosity, Eqs. 13/14 with the sign of reading A9 */
      double vr = 0.0;
      for (int c = 0; c < 3; ++c) vr += (u[3 * i + c] - u[3 * j + c]) * xij[c];
      if (s->P.visc_mode == OC_VISC_BILATERAL || vr < 0.0) {
        const double rho_bar = 0.5 * (rho[i] + rho[j]);
        const double coef = av * (m / rho_bar) * vr / (r2 + s->xi2);
        for (int c = 0; c < 3; ++c) Pi[c] += coef * gW[c];
      }
    }
    o[0] = is_fluid ? -rho[i] * cont : 0.0;
    for (int c = 0; c < 3; ++c) o[1 + c] = mom[c] / rho[i] + (is_fluid ? s->P.gravity[c] : 0.0) + Pi[c];
    if (is_fluid) oc_stress_rate(L, &sig[6 * i], s->P.K, s->P.G, &o[4]);
  }
}

static int check_finite(oc_sim* s) {
  for (int64_t i = 0; i < s->n; ++i) {
    if (s->kind[i] != OC_FLUID) continue;
    int ok = isfinite(s->rho[i]);
    for (int c = 0; c < 3; ++c) ok &= isfinite(s->x[3 * i + c]) && isfinite(s->u[3 * i + c]);
    for (int c = 0; c < 6; ++c) ok &= isfinite(s->sig[6 * i + c]);
    if (!ok) {
      snprintf(s->err, sizeof s->err, "non-finite state at particle id %lld after step %lld",
               (long long)i, (long long)s->steps_done);
      return OC_E_NONFINITE;
    }
  }
  return OC_OK;
}

/* One explicit-midpoint RK2 step with the return map. */
static int step_once(oc_sim* s, double dt) {
  const int64_t n = s->n;
  int rc;
  /* Alg. 2: "if t mod ps_freq = 0: rebuild neighbor lists based on current positions";
   * otherwise the (potentially stale) lists of the last rebuild are used as they are.
   * Both RK stages use the same lists (A17). */
  const int ps_freq = s->P.ps_freq > 0 ? s->P.ps_freq : 1;
  structure_t* kept = (structure_t*)s->kept;
  if (!kept || s->steps_done % ps_freq == 0) {
    if (!kept) {
      kept = (structure_t*)calloc(1, sizeof(structure_t));
      if (!kept) return OC_E_OOM;
      s->kept = kept;
    } else {
      free_structure(kept);
    }
    /* Alg. 3 steps 1–3: flags from the active boxes at t_n, refreshed with the lists (A30) */
    if ((rc = build_structure(s, s->x, kept, 1, compute_activity(s))) != OC_OK) {
      free(kept);
      s->kept = NULL;
      return rc;
    }
  }
  const structure_t st = *kept;
  double* xm = (double*)malloc((size_t)n * 3 * sizeof(double));
  double* um = (double*)malloc((size_t)n * 3 * sizeof(double));
  double* rm = (double*)malloc((size_t)n * sizeof(double));
  double* sm = (double*)malloc((size_t)n * 6 * sizeof(double));
  double* ub = (double*)malloc((size_t)n * 3 * sizeof(double));
  double* ab = (double*)malloc((size_t)n * 3 * sizeof(double));
  if (!xm || !um || !rm || !sm || !ub || !ab) { rc = OC_E_OOM; goto done; }
  pose_t poses[OC_MAX_BODIES];

  /* ---- stage A at y_n ---- */
  for (int b = 0; b < s->nb; ++b) body_pose(&s->bodies[b], 0.0, &poses[b]);
  for (int64_t i = 0; i < n; ++i)
    if (s->kind[i] == OC_BCE) { double xw[3]; marker_kinematics(s, poses, i, xw, &ub[3 * i], &ab[3 * i]); }
  {
    double* bu = (double*)malloc((size_t)n * 3 * sizeof(double));
    double* bs = (double*)malloc((size_t)n * 6 * sizeof(double));
    if (!bu || !bs) { free(bu); free(bs); rc = OC_E_OOM; goto done; }
    bce_extrapolate(s, &st, s->x, s->u, s->rho, s->sig, ub, ab, bu, bs);
    for (int64_t i = 0; i < n; ++i)
      if (s->kind[i] == OC_BCE) {
        for (int c = 0; c < 3; ++c) s->u[3 * i + c] = bu[3 * i + c];
        for (int c = 0; c < 6; ++c) s->sig[6 * i + c] = bs[6 * i + c];
        s->rho[i] = s->P.rho0;
      }
    free(bu); free(bs);
  }
  for (int64_t i = 0; i < n; ++i) {
    double* d = &s->bce[0][9 * i];
    for (int c = 0; c < 3; ++c) d[c] = s->u[3 * i + c];
    for (int c = 0; c < 6; ++c) d[3 + c] = s->sig[6 * i + c];
  }
  rates(s, &st, s->x, s->u, s->rho, s->sig, s->rates[0]);
  /* y_mid = y_n + dt/2 f(t_n, y_n) for fluid; markers follow their body to t_n + dt/2 */
  for (int b = 0; b < s->nb; ++b) body_pose(&s->bodies[b], 0.5 * dt, &poses[b]);
  for (int64_t i = 0; i < n; ++i) {
    const double* f = &s->rates[0][10 * i];
    if (s->kind[i] == OC_FLUID) {
      const double hx = frozen(&st, i) ? 0.0 : 0.5 * dt;   /* A31: a frozen particle stays put */
      for (int c = 0; c < 3; ++c) {
        xm[3 * i + c] = s->x[3 * i + c] + hx * s->u[3 * i + c];
        um[3 * i + c] = s->u[3 * i + c] + 0.5 * dt * f[1 + c];
      }
      rm[i] = s->rho[i] + 0.5 * dt * f[0];
      for (int c = 0; c < 6; ++c) sm[6 * i + c] = s->sig[6 * i + c] + 0.5 * dt * f[4 + c];
    } else {
      marker_kinematics(s, poses, i, &xm[3 * i], &ub[3 * i], &ab[3 * i]);
      for (int c = 0; c < 3; ++c) um[3 * i + c] = s->u[3 * i + c];
      rm[i] = s->P.rho0;
      for (int c = 0; c < 6; ++c) sm[6 * i + c] = s->sig[6 * i + c];
    }
  }

  /* ---- stage B at y_mid (BCE re-extrapolated, A14) ---- */
  {
    double* bu = (double*)malloc((size_t)n * 3 * sizeof(double));
    double* bs = (double*)malloc((size_t)n * 6 * sizeof(double));
    if (!bu || !bs) { free(bu); free(bs); rc = OC_E_OOM; goto done; }
    bce_extrapolate(s, &st, xm, um, rm, sm, ub, ab, bu, bs);
    for (int64_t i = 0; i < n; ++i)
      if (s->kind[i] == OC_BCE) {
        for (int c = 0; c < 3; ++c) um[3 * i + c] = bu[3 * i + c];
        for (int c = 0; c < 6; ++c) sm[6 * i + c] = bs[6 * i + c];
      }
    free(bu); free(bs);
  }
  for (int64_t i = 0; i < n; ++i) {
    double* d = &s->bce[1][9 * i];
    for (int c = 0; c < 3; ++c) d[c] = um[3 * i + c];
    for (int c = 0; c < 6; ++c) d[3 + c] = sm[6 * i + c];
  }
  rates(s, &st, xm, um, rm, sm, s->rates[1]);

  /* ---- y_{n+1} = y_n + dt f(t_n + dt/2, y_mid), then the return map on sigma* ---- */
  #pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    if (s->kind[i] != OC_FLUID || frozen(&st, i)) continue;     /* Extended/Inactive: frozen (A31) */
    const double* f = &s->rates[1][10 * i];
    double sig_star[6], sig_new[6];
    for (int c = 0; c < 3; ++c) {
      s->x[3 * i + c] += dt * um[3 * i + c];
      s->u[3 * i + c] += dt * f[1 + c];
    }
    s->rho[i] += dt * f[0];
    for (int c = 0; c < 6; ++c) sig_star[c] = s->sig[6 * i + c] + dt * f[4 + c];
    oc_return_map(sig_star, &s->sig[6 * i], &s->P, dt, sig_new);
    for (int c = 0; c < 6; ++c) s->sig[6 * i + c] = sig_new[c];
  }
  /* markers keep the stage-B extrapolated u, sigma */
  for (int64_t i = 0; i < n; ++i)
    if (s->kind[i] == OC_BCE) {
      for (int c = 0; c < 3; ++c) s->u[3 * i + c] = um[3 * i + c];
      for (int c = 0; c < 6; ++c) s->sig[6 * i + c] = sm[6 * i + c];
    }

  /* ---- bodies: loads from stage-B marker accelerations (A13), rigid update ---- */
  for (int b = 1; b < s->nb; ++b) {
    body_rec* r = &s->bodies[b];
    double F[3] = {0, 0, 0}, T[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i) {
      if (s->kind[i] != OC_BCE || s->body[i] != b) continue;
      const double* f = &s->rates[1][10 * i];
      double fi[3], rr[3], t[3];
      for (int c = 0; c < 3; ++c) { fi[c] = s->m * f[1 + c]; rr[c] = xm[3 * i + c] - poses[b].pos[c]; }
      cross(rr, fi, t);
      for (int c = 0; c < 3; ++c) { F[c] += fi[c]; T[c] += t[c]; }
    }
    for (int c = 0; c < 3; ++c) { r->force[c] = F[c]; r->torque[c] = T[c]; }
    if (r->b.motion == OC_BODY_FREE) {
      /* semi-implicit Euler (the multibody engine itself is out of scope).  Rotation by
       * Euler's equations in the body's principal frame (inertia = principal moments about the
       * body axes): I alpha_b = T_b - omega_b x (I omega_b), with T_b = R^T T, omega_b = R^T omega
       * at t_n, and alpha = R alpha_b; the DOF mask locks world axes (a locked axis keeps its
       * omega component). */
      double Rb[9], wb[3], Tb[3], Iw[3], gyro[3], ab[3];
      quat_to_R(r->b.quat, Rb);
      for (int a = 0; a < 3; ++a) {
        wb[a] = Rb[a] * r->b.omega[0] + Rb[3 + a] * r->b.omega[1] + Rb[6 + a] * r->b.omega[2];
        Tb[a] = Rb[a] * T[0] + Rb[3 + a] * T[1] + Rb[6 + a] * T[2];
      }
      for (int a = 0; a < 3; ++a) Iw[a] = r->b.inertia[a] * wb[a];
      cross(wb, Iw, gyro);
      for (int a = 0; a < 3; ++a) ab[a] = r->b.inertia[a] > 0 ? (Tb[a] - gyro[a]) / r->b.inertia[a] : 0.0;
      for (int c = 0; c < 3; ++c) {
        const int tfree = (r->b.dof_mask >> c) & 1, rfree = (r->b.dof_mask >> (3 + c)) & 1;
        r->acc[c] = tfree ? F[c] / r->b.mass + s->P.gravity[c] : 0.0;
        r->alpha[c] = rfree ? Rb[3 * c] * ab[0] + Rb[3 * c + 1] * ab[1] + Rb[3 * c + 2] * ab[2] : 0.0;
        r->b.vel[c] += dt * r->acc[c];
        r->b.omega[c] += dt * r->alpha[c];
        r->b.pos[c] += dt * r->b.vel[c];
      }
      quat_advance(r->b.quat, r->b.omega, dt);
    } else if (r->b.motion == OC_BODY_PRESCRIBED) {
      for (int c = 0; c < 3; ++c) { r->b.pos[c] += dt * r->b.vel[c]; r->acc[c] = 0; r->alpha[c] = 0; }
      quat_advance(r->b.quat, r->b.omega, dt);
    }
  }
  for (int b = 0; b < s->nb; ++b) body_pose(&s->bodies[b], 0.0, &poses[b]);
  for (int64_t i = 0; i < n; ++i)
    if (s->kind[i] == OC_BCE && s->bodies[s->body[i]].b.motion != OC_BODY_FIXED) {
      double ubb[3], abb[3];
      marker_kinematics(s, poses, i, &s->x[3 * i], ubb, abb);
    }
  s->steps_done++;
  s->time += dt;
  rc = check_finite(s);
done:
  free(xm); free(um); free(rm); free(sm); free(ub); free(ab);
  return rc;
}

int oc_step(oc_sim* s, double dt, int64_t nsteps) {
  if (!(dt > 0) || nsteps < 0) return OC_E_INVALID;
  for (int64_t k = 0; k < nsteps; ++k) {
    int rc = step_once(s, dt);
    if (rc) return rc;
  }
  return OC_OK;
}

int oc_get_state(const oc_sim* s, int64_t first, int64_t count, double* pos, double* vel,
                 double* rho, double* sig6) {
  if (first < 0 || count < 0 || first + count > s->n) return OC_E_INVALID;
  for (int64_t k = 0; k < count; ++k) {
    const int64_t i = first + k;
    for (int c = 0; c < 3; ++c) {
      if (pos) pos[3 * k + c] = s->x[3 * i + c];
      if (vel) vel[3 * k + c] = s->u[3 * i + c];
    }
    if (rho) rho[k] = s->rho[i];
    if (sig6) for (int c = 0; c < 6; ++c) sig6[6 * k + c] = s->sig[6 * i + c];
  }
  return OC_OK;
}

int oc_set_state(oc_sim* s, int64_t first, int64_t count, const double* pos, const double* vel,
                 const double* rho, const double* sig6) {
  if (first < 0 || count < 0 || first + count > s->n) return OC_E_INVALID;
  for (int64_t k = 0; k < count; ++k) {
    const int64_t i = first + k;
    if (s->kind[i] == OC_BCE && s->bodies[s->body[i]].b.motion != OC_BODY_FIXED && pos)
      return OC_E_INVALID;   /* moving markers follow their body */
    for (int c = 0; c < 3; ++c) {
      if (pos) { s->x[3 * i + c] = pos[3 * k + c]; if (s->kind[i] == OC_BCE) s->xl[3 * i + c] = pos[3 * k + c]; }
      if (vel) s->u[3 * i + c] = vel[3 * k + c];
    }
    if (rho && s->kind[i] == OC_FLUID) s->rho[i] = rho[k];
    if (sig6) for (int c = 0; c < 6; ++c) s->sig[6 * i + c] = sig6[6 * k + c];
  }
  if (pos) drop_kept(s);   /* positions changed: the next step rebuilds the lists */
  return OC_OK;
}

int oc_get_body(const oc_sim* s, int32_t body, oc_body* state, double force[3], double torque[3]) {
  if (body < 0 || body >= s->nb) return OC_E_INVALID;
  if (state) *state = s->bodies[body].b;
  for (int c = 0; c < 3; ++c) {
    if (force) force[c] = s->bodies[body].force[c];
    if (torque) torque[c] = s->bodies[body].torque[c];
  }
  return OC_OK;
}

int oc_last_rates(const oc_sim* s, int stage, double* drho, double* acc, double* dsig6) {
  if (stage < 0 || stage > 1 || s->steps_done == 0) return OC_E_STATE;
  for (int64_t i = 0; i < s->n; ++i) {
    const double* o = &s->rates[stage][10 * i];
    if (drho) drho[i] = o[0];
    for (int c = 0; c < 3; ++c) if (acc) acc[3 * i + c] = o[1 + c];
    for (int c = 0; c < 6; ++c) if (dsig6) dsig6[6 * i + c] = o[4 + c];
  }
  return OC_OK;
}

int oc_last_bce(const oc_sim* s, int stage, double* vel, double* sig6) {
  if (stage < 0 || stage > 1 || s->steps_done == 0) return OC_E_STATE;
  for (int64_t i = 0; i < s->n; ++i) {
    const double* d = &s->bce[stage][9 * i];
    for (int c = 0; c < 3; ++c) if (vel) vel[3 * i + c] = d[c];
    for (int c = 0; c < 6; ++c) if (sig6) sig6[6 * i + c] = d[3 + c];
  }
  return OC_OK;
}

const char* oc_last_error(const oc_sim* s) { return s ? s->err : ""; }

int oc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* thread count of the following parallel loops (timing the oracle on 1 core; no arithmetic effect:
   every loop is a gather with per-particle results) */
void oc_set_num_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
