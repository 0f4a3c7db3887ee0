// physics.cuh — BCE extrapolation, fused rates + RK2 epilogues + return map, rigid bodies.
//
//   k_body_poses  body kinematics at t_n and t_n + dt/2 (markers follow their body)
//   k_bce         Adami extrapolation of u, sigma onto every marker (A11, A12)
//   k_rates<0>    stage A: rates at y_n -> y_mid = y_n + dt/2 f
//   k_rates<1>    stage B: rates at y_mid with the same lists -> y_{n+1} = y_n + dt f,
//                 mu(I) return map; marker accelerations of moving bodies (A13)
//   k_body_update deterministic fp64 reduction of marker loads, semi-implicit Euler
#pragma once
#include "common.cuh"

namespace crmk {

// ------------------------------------------------------------------------------------
__device__ __forceinline__ void quat_advance_d(double q[4], const double w[3], double tau) {
  const double wn = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
  if (wn == 0.0) return;
  const double ang = 0.5 * wn * tau, c = cos(ang), sn = sin(ang) / wn;
  const double d[4] = {c, sn * w[0], sn * w[1], sn * w[2]};
  const double r[4] = {d[0] * q[0] - d[1] * q[1] - d[2] * q[2] - d[3] * q[3],
                       d[0] * q[1] + d[1] * q[0] + d[2] * q[3] - d[3] * q[2],
                       d[0] * q[2] - d[1] * q[3] + d[2] * q[0] + d[3] * q[1],
                       d[0] * q[3] + d[1] * q[2] - d[2] * q[1] + d[3] * q[0]};
  const double nn = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2] + r[3] * r[3]);
  for (int k = 0; k < 4; ++k) q[k] = r[k] / nn;
}

// unit quaternion (w, x, y, z) -> rotation matrix (row-major, body -> world)
__device__ __forceinline__ void quat_R_d(const double q[4], double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

__device__ __forceinline__ void make_pose(const BodyState& b, double tau, Pose& out) {
  double q[4] = {b.quat[0], b.quat[1], b.quat[2], b.quat[3]};
  quat_advance_d(q, b.omega, tau);
  double R[9];
  quat_R_d(q, R);
  for (int k = 0; k < 9; ++k) out.R[k] = (float)R[k];
  for (int a = 0; a < 3; ++a) {
    out.pos[a] = (float)(b.pos[a] + tau * b.vel[a]);
    out.vel[a] = (float)b.vel[a];
    out.omega[a] = (float)b.omega[a];
    out.acc[a] = (float)b.acc[a];
    out.alpha[a] = (float)b.alpha[a];
  }
}

__global__ void k_body_poses(int nb, const BodyState* __restrict__ bodies, double half_dt,
                             Pose* __restrict__ pose0, Pose* __restrict__ pose_mid) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  make_pose(bodies[b], 0.0, pose0[b]);
  make_pose(bodies[b], half_dt, pose_mid[b]);
}

__device__ __forceinline__ void body_kinematics(const Pose& q, float x, float y, float z, float ub[3], float ab[3]) {
  const float r[3] = {x - q.pos[0], y - q.pos[1], z - q.pos[2]};
  const float* w = q.omega;
  const float wr[3] = {w[1] * r[2] - w[2] * r[1], w[2] * r[0] - w[0] * r[2], w[0] * r[1] - w[1] * r[0]};
  const float wwr[3] = {w[1] * wr[2] - w[2] * wr[1], w[2] * wr[0] - w[0] * wr[2], w[0] * wr[1] - w[1] * wr[0]};
  const float* al = q.alpha;
  const float ar[3] = {al[1] * r[2] - al[2] * r[1], al[2] * r[0] - al[0] * r[2], al[0] * r[1] - al[1] * r[0]};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ub[a] = q.vel[a] + wr[a];
    ab[a] = q.acc[a] + ar[a] + wwr[a];
  }
}

// ------------------------------------------------------------------------------------
// mu(I) return map in fp32; readings A16 (gamma_dot >= 0, p floor 1 Pa for I
// only, I = 0 -> mu_s), A27 (tau_max >= 0).  s, sn = (xx,yy,zz,xy,xz,yz)
__device__ __forceinline__ void return_map(float s[6], const float sn[6], const Phys& ph, float dt) {
  const float p = -(s[0] + s[1] + s[2]) * (1.0f / 3.0f);
  const float t0 = s[0] + p, t1 = s[1] + p, t2 = s[2] + p;
  const float tb = sqrtf(0.5f * (t0 * t0 + t1 * t1 + t2 * t2) + (s[3] * s[3] + s[4] * s[4] + s[5] * s[5]));
  const float p_cri = -ph.coh / ph.mu_s;
  if (p < p_cri) {   // Step 1
#pragma unroll
    for (int k = 0; k < 6; ++k) s[k] = 0.f;
    return;
  }
  const float pn = -(sn[0] + sn[1] + sn[2]) * (1.0f / 3.0f);
  const float n0 = sn[0] + pn, n1 = sn[1] + pn, n2 = sn[2] + pn;
  const float tbn = sqrtf(0.5f * (n0 * n0 + n1 * n1 + n2 * n2) + (sn[3] * sn[3] + sn[4] * sn[4] + sn[5] * sn[5]));
  const float gd = fmaxf(0.f, (tb - tbn) / (ph.G * dt));                 // Step 2
  const float I = gd * ph.grain_d * sqrtf(ph.rho0 / fmaxf(p, 1.0f));
  const float mu = (I > 0.f) ? ph.mu_s + (ph.mu_2 - ph.mu_s) / (1.0f + ph.I0 / I) : ph.mu_s;
  const float tmax = fmaxf(mu * p + ph.coh, 0.f);                          // Step 3
  if (tb <= tmax) return;
  const float sc = tmax / tb;                                             // Step 4
  s[0] = sc * t0 - p; s[1] = sc * t1 - p; s[2] = sc * t2 - p;
  s[3] *= sc; s[4] *= sc; s[5] *= sc;
}

// ------------------------------------------------------------------------------------
// Loads of moving bodies (A13) from the stage-B marker accelerations: a deterministic
// fixed-order fp64 reduction over this rank's markers (k_body_partial, one block per moving body),
// then — after the slabs exchanged their partial sums (multi-GPU) — the sum over ranks in rank order
// and the rigid update (semi-implicit Euler, once per step; k_body_integrate).
constexpr int BODY_BS = 256;
__global__ void __launch_bounds__(BODY_BS) k_body_partial(const int* __restrict__ moving_bodies,
                                                          const uint32_t* __restrict__ mstart,
                                                          const uint32_t* __restrict__ moving_ids,
                                                          const uint32_t* __restrict__ slot_of_id,
                                                          const float4* __restrict__ U,
                                                          const float4* __restrict__ macc,
                                                          const float4* __restrict__ Pmid,
                                                          const float4* __restrict__ Lmid,
                                                          const BodyState* __restrict__ bodies, double dt,
                                                          double* __restrict__ partial) {
  __shared__ double red[6][BODY_BS];
  const int bi = blockIdx.x;
  const BodyState& B = bodies[moving_bodies[bi]];
  const double pm[3] = {B.pos[0] + 0.5 * dt * B.vel[0], B.pos[1] + 0.5 * dt * B.vel[1], B.pos[2] + 0.5 * dt * B.vel[2]};
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (uint32_t k = mstart[bi] + threadIdx.x; k < mstart[bi + 1]; k += BODY_BS) {
    const uint32_t s = slot_of_id[moving_ids[k]];
    if (s == 0xffffffffu || tag_ghost(tag_of(U[s].w))) continue;   // owned by another slab
    const float4 f = macc[s];
    const float4 x = Pmid[s], xl = Lmid[s];
    const double r[3] = {(double)x.x + (double)xl.x - pm[0], (double)x.y + (double)xl.y - pm[1],
                         (double)x.z + (double)xl.z - pm[2]};
    const double fx = f.x, fy = f.y, fz = f.z;
    acc[0] += fx; acc[1] += fy; acc[2] += fz;
    acc[3] += r[1] * fz - r[2] * fy;
    acc[4] += r[2] * fx - r[0] * fz;
    acc[5] += r[0] * fy - r[1] * fx;
  }
  for (int c = 0; c < 6; ++c) red[c][threadIdx.x] = acc[c];
  __syncthreads();
  for (int o = BODY_BS / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int c = 0; c < 6; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x < 6) partial[bi * 6 + threadIdx.x] = red[threadIdx.x][0];
}

// parts: world blocks of nbm x 6 partial sums (rank order); one thread per moving body
__global__ void k_body_integrate(int nbm, const int* __restrict__ moving_bodies, const double* __restrict__ parts,
                                 int world, BodyState* __restrict__ bodies, double dt, double g0, double g1, double g2,
                                 const ErrLatch* err) {
  const int bi = blockIdx.x * blockDim.x + threadIdx.x;
  if (bi >= nbm || latched(err)) return;
  BodyState& B = bodies[moving_bodies[bi]];
  double F[3], T[3];
  for (int c = 0; c < 3; ++c) { F[c] = parts[bi * 6 + c]; T[c] = parts[bi * 6 + 3 + c]; }
  for (int r = 1; r < world; ++r)
    for (int c = 0; c < 3; ++c) {
      F[c] += parts[(size_t)r * nbm * 6 + bi * 6 + c];
      T[c] += parts[(size_t)r * nbm * 6 + bi * 6 + 3 + c];
    }
  const double g[3] = {g0, g1, g2};
  for (int c = 0; c < 3; ++c) { B.force[c] = F[c]; B.torque[c] = T[c]; }
  if (B.motion == 1) {   // FREE
    // rotation by Euler's equations in the principal (body) frame at t_n:
    // I alpha_b = T_b - omega_b x (I omega_b), T_b = R^T T, omega_b = R^T omega, alpha = R alpha_b;
    // the DOF mask locks world axes
    double R[9];
    quat_R_d(B.quat, R);
    double wb[3], Tb[3], ab[3];
    for (int a = 0; a < 3; ++a) {
      wb[a] = R[a] * B.omega[0] + R[3 + a] * B.omega[1] + R[6 + a] * B.omega[2];
      Tb[a] = R[a] * T[0] + R[3 + a] * T[1] + R[6 + a] * T[2];
    }
    const double Iw[3] = {B.inertia[0] * wb[0], B.inertia[1] * wb[1], B.inertia[2] * wb[2]};
    const double gy[3] = {wb[1] * Iw[2] - wb[2] * Iw[1], wb[2] * Iw[0] - wb[0] * Iw[2], wb[0] * Iw[1] - wb[1] * Iw[0]};
    for (int a = 0; a < 3; ++a) ab[a] = B.inertia[a] > 0 ? (Tb[a] - gy[a]) / B.inertia[a] : 0.0;
    for (int c = 0; c < 3; ++c) {
      const int tfree = (B.dof_mask >> c) & 1, rfree = (B.dof_mask >> (3 + c)) & 1;
      B.acc[c] = tfree ? F[c] / B.mass + g[c] : 0.0;
      B.alpha[c] = rfree ? R[3 * c] * ab[0] + R[3 * c + 1] * ab[1] + R[3 * c + 2] * ab[2] : 0.0;
      B.vel[c] += dt * B.acc[c];
      B.omega[c] += dt * B.alpha[c];
      B.pos[c] += dt * B.vel[c];
    }
    quat_advance_d(B.quat, B.omega, dt);
  } else if (B.motion == 2) {   // PRESCRIBED
    for (int c = 0; c < 3; ++c) { B.pos[c] += dt * B.vel[c]; B.acc[c] = 0; B.alpha[c] = 0; }
    quat_advance_d(B.quat, B.omega, dt);
  }
}

// ------------------------------------------------------------------------------------
// state <-> fp64 id-order staging (crm_get_state / crm_set_state)
__global__ void k_get_state(long long first, long long count, const uint32_t* __restrict__ slot_of_id,
                            const float4* __restrict__ P, const float4* __restrict__ L,
                            const float4* __restrict__ U, const float4* __restrict__ S1,
                            const float2* __restrict__ S2, double* __restrict__ pos, double* __restrict__ vel,
                            double* __restrict__ rho, double* __restrict__ sig) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const uint32_t s = slot_of_id[first + k];
  if (s == 0xffffffffu) return;                 // not on this rank (multi-GPU): row left as is
  const float4 p = P[s], u = U[s], s1 = S1[s];
  if (tag_ghost(tag_of(u.w))) return;           // ghost copy: owned by a neighbour slab
  const float2 s2 = S2[s];
  const float4 l = L[s];
  pos[3 * k] = (double)p.x + (double)l.x;       // compensated position hi + lo
  pos[3 * k + 1] = (double)p.y + (double)l.y;
  pos[3 * k + 2] = (double)p.z + (double)l.z;
  vel[3 * k] = u.x; vel[3 * k + 1] = u.y; vel[3 * k + 2] = u.z;
  rho[k] = p.w;
  sig[6 * k] = s1.x; sig[6 * k + 1] = s1.y; sig[6 * k + 2] = s1.z;
  sig[6 * k + 3] = s1.w; sig[6 * k + 4] = s2.x; sig[6 * k + 5] = s2.y;
}

__global__ void k_set_state(long long first, long long count, const uint32_t* __restrict__ slot_of_id,
                            float4* __restrict__ P, float4* __restrict__ L, float4* __restrict__ U,
                            float4* __restrict__ S1, float2* __restrict__ S2, const double* __restrict__ pos,
                            const double* __restrict__ vel, const double* __restrict__ rho,
                            const double* __restrict__ sig, int has_pos, int has_vel, int has_rho, int has_sig) {
  const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const uint32_t s = slot_of_id[first + k];
  if (s == 0xffffffffu) return;
  float4 p = P[s], u = U[s];
  if (tag_ghost(tag_of(u.w))) return;
  if (has_pos) {   // hi = fp32 rounding of x (what rules B1/B2 see), lo = the remainder
    p.x = (float)pos[3 * k]; p.y = (float)pos[3 * k + 1]; p.z = (float)pos[3 * k + 2];
    const float4 l = make_float4((float)(pos[3 * k] - (double)p.x), (float)(pos[3 * k + 1] - (double)p.y),
                                 (float)(pos[3 * k + 2] - (double)p.z), 0.f);
    L[s] = l;
    u.w = __uint_as_float(tag_with_lo(tag_of(u.w), p.x, p.y, p.z, l.x, l.y, l.z));
  }
  if (has_rho && !tag_is_bce(tag_of(u.w))) p.w = (float)rho[k];
  if (has_vel) { u.x = (float)vel[3 * k]; u.y = (float)vel[3 * k + 1]; u.z = (float)vel[3 * k + 2]; }
  P[s] = p;
  U[s] = u;
  if (has_sig) {
    S1[s] = make_float4((float)sig[6 * k], (float)sig[6 * k + 1], (float)sig[6 * k + 2], (float)sig[6 * k + 3]);
    S2[s] = make_float2((float)sig[6 * k + 4], (float)sig[6 * k + 5]);
  }
}

}  // namespace crmk
