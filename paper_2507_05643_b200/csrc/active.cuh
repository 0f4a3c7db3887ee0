// active.cuh — active domains (Alg. 3).
//
//   k_activity  UpdateActivity + ComputeActiveCount: one flag per particle from the active
//               boxes (OOBBs at the bodies' local origins) at the pose of the step start;
//               warp-aggregated counts of Active / Extended-Active / Inactive.
// Inactive particles then get the sentinel key M in k_bin: they sort behind every cell (the active
// set is the prefix [0, N_{a+e}) of the sorted arrays), take no part in the neighbour search and
// are not touched by the tile kernels, so their state stays frozen until a box reaches them again.
// Extended-Active particles carry TAG_FROZEN (reading A31): they are staged, searched and serve as
// neighbours of Active ones ("to ensure their data is available"), but their own state —
// fluid y, marker u and sigma — is not updated ("their states are not updated").
#pragma once
#include <cmath>
#include "common.cuh"

namespace crmk {

constexpr uint8_t ACT_ACTIVE = 0, ACT_EXTENDED = 1, ACT_INACTIVE = 2;

struct ActiveBox {
  double half[3];   // half extents in the body frame
  int body;
  int pad;
};

// A29 / B6: Active inside the box (|x_local| <= half), Extended-Active outside every box but at a
// Euclidean distance < 2h from one, else Inactive; fp64 on the compensated position hi + lo.
// Markers of moving bodies are always Active.
__global__ void k_activity(int n, const float4* __restrict__ P, const float4* __restrict__ L,
                           float4* __restrict__ U, const uint32_t* __restrict__ ids,
                           const BodyState* __restrict__ bodies, const ActiveBox* __restrict__ boxes, int nbox,
                           double radius, uint8_t* __restrict__ act_slot, uint8_t* __restrict__ act_id,
                           unsigned long long* __restrict__ counts, const uint32_t* __restrict__ dn) {
  if (dn) n = (int)*dn;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int f = 3;   // no particle (tail lanes)
  if (i < n) {
    const uint32_t tag = tag_of(U[i].w);
    if (tag_is_bce(tag) && tag_moving(tag)) {
      f = ACT_ACTIVE;
    } else {
      const float4 p = P[i], l = L[i];
      const double x[3] = {(double)p.x + (double)l.x, (double)p.y + (double)l.y, (double)p.z + (double)l.z};
      f = ACT_INACTIVE;
      for (int k = 0; k < nbox; ++k) {
        const ActiveBox bx = boxes[k];
        const BodyState& B = bodies[bx.body];
        const double w = B.quat[0], qx = B.quat[1], qy = B.quat[2], qz = B.quat[3];
        // columns of the body->world rotation: the body axes in world coordinates
        const double ex[3] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy + w * qz), 2 * (qx * qz - w * qy)};
        const double ey[3] = {2 * (qx * qy - w * qz), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz + w * qx)};
        const double ez[3] = {2 * (qx * qz + w * qy), 2 * (qy * qz - w * qx), 1 - 2 * (qx * qx + qy * qy)};
        const double d[3] = {x[0] - B.pos[0], x[1] - B.pos[1], x[2] - B.pos[2]};
        const double loc[3] = {ex[0] * d[0] + ex[1] * d[1] + ex[2] * d[2], ey[0] * d[0] + ey[1] * d[1] + ey[2] * d[2],
                               ez[0] * d[0] + ez[1] * d[1] + ez[2] * d[2]};
        double dist2 = 0.0;
        bool inside = true;
        for (int a = 0; a < 3; ++a) {
          const double o = fabs(loc[a]) - bx.half[a];
          if (o > 0.0) {
            inside = false;
            dist2 += o * o;
          }
        }
        if (inside) {
          f = ACT_ACTIVE;
          break;
        }
        if (dist2 < radius * radius) f = ACT_EXTENDED;
      }
    }
    act_slot[i] = (uint8_t)f;
    act_id[ids[i]] = (uint8_t)f;
    float4 u = U[i];
    const uint32_t t2 = f == ACT_EXTENDED ? (tag | TAG_FROZEN) : (tag & ~TAG_FROZEN);
    if (t2 != tag) {
      u.w = __uint_as_float(t2);
      U[i] = u;
    }
  }
  // ComputeActiveCount: warp-aggregated
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int v = 0; v < 3; ++v) {
    const unsigned c = __popc(__ballot_sync(0xffffffffu, f == v));
    if (lane == 0 && c) atomicAdd(&counts[v], (unsigned long long)c);
  }
}

// ManageArrayMemory policy: grow to ceil(N G) when N exceeds the capacity; every S_I steps,
// shrink to N when N / capacity < S; otherwise keep.  Host function (the arrays it sizes are
// reallocated by the caller).
inline int64_t manage_capacity(int64_t capacity, int64_t required, int64_t step, double growth, double shrink,
                               int interval, int* action) {
  int a = 0;
  int64_t cap = capacity;
  if (required > capacity) {
    a = 1;
    cap = (int64_t)std::ceil((double)required * growth);
  } else if (interval > 0 && step % interval == 0 && capacity > 0 && (double)required / (double)capacity < shrink) {
    a = 2;
    cap = required;
  }
  if (action) *action = a;
  return cap;
}

}  // namespace crmk
