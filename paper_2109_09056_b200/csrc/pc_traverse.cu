// Consumers of the device neighbor traversal (include/particula_b200_traverse.cuh,
// SURVEY §8 f4): a pair functor (coordination number within r_inner) and a
// three-body functor (per-atom sum of cos(angle j-i-k) over neighbor pairs,
// the building block of angular potentials), each with the Serial and Team
// policies.  Geometry as the reference: dx = x_j - x_i with the exact minimum
// image (pc::min_image), r^2 in the einsum order.
#include "pc_common.cuh"
#include "../../include/particula_b200_traverse.cuh"

namespace pc {

struct MinImage {
  const double* x;
  pc_box b;
  __device__ __forceinline__ void d(int i, int j, double o[3]) const {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o[a] = __dsub_rn(x[3 * (int64_t)j + a], x[3 * (int64_t)i + a]);
      if (b.periodic[a]) o[a] = min_image(o[a], b.length[a], b.mi_thresh[a]);
    }
  }
};

struct Coordination {
  MinImage g;
  double r2max;
  double* out;
  __device__ void operator()(int i, int j) const {
    double d[3];
    g.d(i, j, d);
    if (r2_exact(d[0], d[1], d[2]) < r2max) atomicAdd(out + i, 1.0);
  }
};

struct AngleSum {
  MinImage g;
  double* out;
  __device__ void operator()(int i, int j, int k) const {
    double u[3], w[3];
    g.d(i, j, u);
    g.d(i, k, w);
    const double uu = r2_exact(u[0], u[1], u[2]), ww = r2_exact(w[0], w[1], w[2]);
    const double uw = __dadd_rn(__dadd_rn(__dmul_rn(u[0], w[0]), __dmul_rn(u[2], w[2])),
                                __dmul_rn(u[1], w[1]));
    atomicAdd(out + i, __ddiv_rn(uw, __dsqrt_rn(__dmul_rn(uu, ww))));
  }
};

}  // namespace pc

extern "C" {

using namespace pc;

int pc_traverse_coordination(const double* d_x, const pc_box* box, const int64_t* d_offsets,
                             const int32_t* d_index, int32_t n, int32_t begin, int32_t end,
                             double r_inner, int32_t team, double* d_out, void* stream) {
  pc_traverse::CsrList l{d_offsets, d_index, n};
  Coordination f{MinImage{d_x, *box}, r_inner * r_inner, d_out};
  const cudaError_t e = pc_traverse::for_each_neighbor(
      l, begin, end, f, team ? pc_traverse::Policy::Team : pc_traverse::Policy::Serial,
      as_stream(stream));
  if (e != cudaSuccess) {
    set_error("pc_traverse_coordination: %s", cudaGetErrorString(e));
    return PC_ERR_RUNTIME;
  }
  note_launch(1);
  return PC_OK;
}

int pc_traverse_angle_sum(const double* d_x, const pc_box* box, const int64_t* d_offsets,
                          const int32_t* d_index, int32_t n, int32_t begin, int32_t end,
                          int32_t team, double* d_out, void* stream) {
  pc_traverse::CsrList l{d_offsets, d_index, n};
  AngleSum f{MinImage{d_x, *box}, d_out};
  const cudaError_t e = pc_traverse::for_each_neighbor2(
      l, begin, end, f, team ? pc_traverse::Policy::Team : pc_traverse::Policy::Serial,
      as_stream(stream));
  if (e != cudaSuccess) {
    set_error("pc_traverse_angle_sum: %s", cudaGetErrorString(e));
    return PC_ERR_RUNTIME;
  }
  note_launch(1);
  return PC_OK;
}

}  // extern "C"
