// common.cuh — device-side types shared by the libcrm kernels (sm_100a).
//
// Device state layout (HBM, structure of arrays, (cell, id) sorted order):
//   P  float4 (x, y, z, rho)          positions + density          16 B
//   U  float4 (u, v, w, tag)          velocity + kind/body tag      16 B
//   S1 float4 (sxx, syy, szz, sxy)    stress part 1                 16 B
//   S2 float2 (sxz, syz)              stress part 2                  8 B
// i.e. 56 B per particle; fluid and BCE markers share the arrays (A8: markers are
// ordinary neighbours carrying extrapolated u, sigma and rho0).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace crmk {

// tag word stored in U.w (bit pattern, not a float value)
//   bit 0      : 1 = BCE marker, 0 = fluid
//   bits 1..7  : body index (0 = static walls; at most 127 bodies)
//   bit 8      : 1 = the body moves (FREE or PRESCRIBED)
__host__ __device__ __forceinline__ uint32_t make_tag(uint32_t kind, uint32_t body, uint32_t moving) {
  return (kind & 1u) | ((body & 0x7fu) << 1) | ((moving & 1u) << 8);
}
//   bit 9      : ghost copy of a neighbour slab's particle (multi-GPU)
//   bit 10     : dropped at the next sort (migrated to a neighbour slab)
//   bit 11     : Extended-Active particle of Alg. 3 (reading A31): a neighbour only, state frozen
//   bits 12..29: the position's compensation term lo (x = hi + lo) quantised to 6
//                signed bits per axis in units of |hi| 2^-29 (|lo| <= ulp(hi)/2 <= |hi| 2^-24, so
//                the code spans it; resolution <= ulp(hi)/32).  The pair and BCE kernels read it from
//                the staged window (no global lo loads); the integrator keeps the exact lo in L.
//   bits 30,31 : 0 (the word is a finite float bit pattern)
constexpr uint32_t TAG_GHOST = 1u << 9;
constexpr uint32_t TAG_DROP = 1u << 10;
constexpr uint32_t TAG_FROZEN = 1u << 11;
constexpr uint32_t TAG_FLAGS = 0xfffu;   // everything but the quantised lo
__device__ __forceinline__ uint32_t tag_of(float w) { return __float_as_uint(w); }
__device__ __forceinline__ bool tag_is_bce(uint32_t t) { return t & 1u; }
__device__ __forceinline__ uint32_t tag_body(uint32_t t) { return (t >> 1) & 0x7fu; }
__device__ __forceinline__ bool tag_moving(uint32_t t) { return (t >> 8) & 1u; }
__device__ __forceinline__ bool tag_ghost(uint32_t t) { return (t & TAG_GHOST) != 0u; }
__device__ __forceinline__ bool tag_frozen(uint32_t t) { return (t & TAG_FROZEN) != 0u; }

// quantised lo of one axis: 6-bit two's complement code of lo / (|hi| 2^-29)
__host__ __device__ __forceinline__ uint32_t loq_code(float hi, float lo) {
  const float unit = fabsf(hi) * 1.86264514923095703125e-9f;   // |hi| 2^-29
#ifdef __CUDA_ARCH__
  float q = unit > 0.f ? rintf(__fdividef(lo, unit)) : 0.f;   // (an encoding: the approximate quotient is fine)
#else
  float q = unit > 0.f ? rintf(lo / unit) : 0.f;
#endif
  q = fminf(fmaxf(q, -32.f), 31.f);
  return (uint32_t)((int)q) & 63u;
}
__host__ __device__ __forceinline__ uint32_t tag_with_lo(uint32_t tag, float hx, float hy, float hz, float lx, float ly,
                                                         float lz) {
  return (tag & TAG_FLAGS) | (loq_code(hx, lx) << 12) | (loq_code(hy, ly) << 18) | (loq_code(hz, lz) << 24);
}
__device__ __forceinline__ float loq_value(uint32_t tag, int axis, float hi) {
  const int q = ((int)(tag << (14 - 6 * axis))) >> 26;   // sign-extended bits 12 + 6 axis .. + 5
  return (float)q * (fabsf(hi) * 1.86264514923095703125e-9f);
}

// fixed grid (reading A19); cells of size s = support*h
struct Grid {
  float lo[3];
  float s;                 // (float)(support*h), B1
  int dims[3];             // Nx, Ny, Nz
  uint32_t M;              // Nx*Ny*Nz
  float R2;                // (float)((support*h)^2), B2
  float margin;            // conservative slack of the cell-box distance pruning (m)
};

// physical constants of one context, fp32
struct Phys {
  float h, hinv;
  float wnorm;             // 1/(pi h^3)  (cubic spline sigma3, A1)
  float fnorm;             // 1/(pi h^5)  (W'(r)/r prefactor)
  float R2;                // support radius squared (W = 0 beyond, A17)
  float m;                 // particle mass rho0 d0^3
  float rho0;
  float avc;               // gamma_a h c_s (Eq. 13)
  float xi2;               // xi^2 (A10)
  float g[3];              // gravity
  float K, G;              // elastic moduli (Eq. 3)
  float mu_s, mu_2, I0, coh, grain_d;   // mu(I) (Eq. muI)
  int unilateral;          // Eq. 14 switch
  // folded constants of the pair loop
  float kin_a;             // 2.25 fnorm / h      : W'/r = kin_a r + kin_b          (q < 1)
  float kin_b;             // -3 fnorm
  float kout;              // -0.75 h fnorm       : W'/r = kout (2 - q)^2 / r       (1 <= q < 2)
  float c_av;              // 2 m gamma_a h c_s   : AV coefficient numerator (Eq. 13)
  int build_lists;         // stage A filters and stores the lists (rebuild step of Alg. 2)
  // quintic Wendland (A28): W = wd_a t^4 (2q + 1), W'/r = wd_f t^3, t = 1 - q/2
  float wd_a;              // 21 / (16 pi h^3)
  float wd_f;              // -5 wd_a / h^2
};

// kernel selection (template parameter of the tile kernels; CRM_KERNEL_* of include/crm.h)
constexpr int KER_CUBIC = 0;
constexpr int KER_WENDLAND = 1;

// W(r) of the selected kernel, r < 2h (branch-free select for the cubic's two pieces)
template <int KER>
__device__ __forceinline__ float kernel_W(float r, const Phys& ph) {
  const float q = r * ph.hinv;
  if (KER == KER_WENDLAND) {
    const float t = fmaf(-0.5f, q, 1.0f);
    const float t2 = t * t;
    return ph.wd_a * t2 * t2 * fmaf(2.0f, q, 1.0f);
  } else {
    const float tt = 2.0f - q;
    return q < 1.0f ? ph.wnorm * (1.0f - 1.5f * q * q + 0.75f * q * q * q) : ph.wnorm * 0.25f * tt * tt * tt;
  }
}

// W'(r)/r of the selected kernel, r > 0 (0 from 2h on); rinv = 1/r
template <int KER>
__device__ __forceinline__ float kernel_F(float r, float rinv, const Phys& ph) {
  if (KER == KER_WENDLAND) {
    const float t = fmaxf(fmaf(-0.5f * ph.hinv, r, 1.0f), 0.0f);   // 0 beyond 2h (A17)
    return ph.wd_f * t * t * t;
  } else {
    // cubic spline (A1): kin_a r + kin_b for r < h, kout (2 - r/h)^2 / r otherwise; both pieces
    // are evaluated and selected (no branch: the pair loops stay straight-line code)
    const float t = fmaxf(fmaf(-ph.hinv, r, 2.0f), 0.0f);   // 0 beyond 2h (A17)
    const float f_in = fmaf(ph.kin_a, r, ph.kin_b);
    const float f_out = (ph.kout * rinv) * (t * t);
    return (r < ph.h) ? f_in : f_out;
  }
}

// MUFU approximations (no IEEE/denormal wrappers): max rel. error ~2^-22 (rsqrt, rcp)
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed fp32 pairs (element 0 in the low word) on sm_100's FADD2/FMUL2/FFMA2: per element the
// IEEE round-to-nearest result of the scalar instruction, half the issue slots; a scalar operand
// broadcast into both elements costs no instruction (the .F32 operand form)
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long f2_make(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ unsigned long long f2_splat(float a) { return f2_make(a, a); }
__device__ __forceinline__ float f2_lo(unsigned long long v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2_hi(unsigned long long v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// rigid-body kinematics at one instant, used to place markers and extrapolate BCE values
struct Pose {
  float pos[3];
  float R[9];
  float vel[3], omega[3], acc[3], alpha[3];
};

// rigid-body state (fp64, device-resident; updated once per step by k_body_update)
struct BodyState {
  double mass, inertia[3], pos[3], quat[4], vel[3], omega[3];
  double acc[3], alpha[3], force[3], torque[3];
  int motion, dof_mask, pad0, pad1;
};

// first-error latch (written with atomicCAS on `code`).  cur_step is the device's step counter:
// k_step_begin sets it (per-kernel launches) or advances it (a replayed CUDA graph, captured with
// step = -1), and stops advancing once an error is latched, so an error names its real step.  The
// state-writing kernels return at entry once the latch is set: the steps after the first bad one
// compute nothing (the state stays as the failing step left it).
struct ErrLatch {
  int code;
  int pad;
  long long step;
  long long id;
  long long aux;
  long long cur_step;
};

__device__ __forceinline__ void latch_error(ErrLatch* e, int code, long long id, long long step, long long aux) {
  if (atomicCAS(&e->code, 0, code) == 0) {
    e->id = id;
    e->step = step >= 0 ? step : e->cur_step;
    e->aux = aux;
  }
}

// true once an error is latched (read at kernel entry: skip the work of the steps after it)
__device__ __forceinline__ bool latched(const ErrLatch* e) { return *(volatile const int*)&e->code != 0; }

__global__ void k_latch_set_step(ErrLatch* e, long long step) { e->cur_step = step; }

// first kernel of every step: step >= 0 sets the counter, step < 0 (graph replay) advances it
__global__ void k_step_begin(ErrLatch* e, long long step) {
  if (e->code) return;
  e->cur_step = step >= 0 ? step : e->cur_step + 1;
}

// Debug capture buffers (sorted order), written only when armed.
struct Debug {
  float* drho[2];
  float4* acc[2];
  float4* ds1[2];
  float2* ds2[2];
  float4* bu[2];
  float4* bs1[2];
  float2* bs2[2];
};

}  // namespace crmk
