// prep.cu -- K0, the parameter sampler (O1) and the per-image LUT
// builder (O8, O12).  One CTA per image: thread 0 walks the op list drawing
// gate + params from Philox4x32-10 and tracking dims; then 256 threads build
// the composed LUT of each LUT stage in fp64 without FMA contraction.
#include "kernels.cuh"

namespace alb {

// GridDistortion knot displacements of one axis (reading R31, in the
// order DESIGN.md states): factors f_i = 1 + U(lo, hi) from draws j0 + i,
// c_{i+1} = c_i + f_i, e_i = (L-1) c_i / S - (L-1) i / n, e_0 = e_n = 0.
__device__ void grid_knots(const alb_op& o, uint64_t seed, uint32_t gi, int k, int j0, int L,
                           double* e) {
  const int n = o.num_steps;
  double c[ALB_GRID_MAX_STEPS + 1];
  c[0] = 0.0;
  for (int i = 0; i < n; ++i)
    c[i + 1] = __dadd_rn(c[i], __dadd_rn(1.0, urange(o.lo[0], o.hi[0], draw_u(seed, gi, k, j0 + i))));
  const double S = c[n], span = (double)(L - 1);
  e[0] = 0.0;
  e[n] = 0.0;
  for (int i = 1; i < n; ++i)
    e[i] = __dsub_rn(__ddiv_rn(__dmul_rn(span, c[i]), S), __ddiv_rn(__dmul_rn(span, (double)i), (double)n));
}

// gate + params of every slot of image i and the dims each slot sees (the
// walk of DESIGN.md O1, sample_core in kernels.cuh); sp / sf (may be null)
// receive copies for the LUT build
__device__ void sample_image(const PrepArgs& a, int i, double (*sp)[kMaxParams], uint8_t* sf) {
  const uint32_t gi = a.first_image + (uint32_t)i;
  double* prm = a.params + (size_t)i * a.n_ops * kMaxParams;
  uint8_t* fired = a.fired + (size_t)i * a.n_ops;
  int32_t* dims = a.dims + (size_t)i * (a.n_ops + 1) * 2;
  sample_core(a.ops, a.n_ops, a.seed, gi, a.in_desc[i].height, a.in_desc[i].width, prm, fired, dims);
  int g_ord = 0;
  for (int k = 0; k < a.n_ops; ++k) {
    const alb_op& o = a.ops[k];
    if (o.kind == ALB_GRID_DISTORTION && a.grid) {  // x factors: draws 1..n+1, y factors: n+2..2n+2
      double* e = a.grid + ((size_t)i * a.n_grid + g_ord++) * kGridStride;
      grid_knots(o, a.seed, gi, k, 1, dims[2 * k + 1], e);
      grid_knots(o, a.seed, gi, k, o.num_steps + 2, dims[2 * k], e + kGridAxis);
    }
    if (sp) {
#pragma unroll
      for (int j = 0; j < kMaxParams; ++j) sp[k][j] = prm[(size_t)k * kMaxParams + j];
    }
    if (sf) sf[k] = fired[k];
  }
}

__global__ void __launch_bounds__(256) k_prep(PrepArgs a) {
  const int i = a.img0 + blockIdx.x;
  __shared__ double s_prm[kMaxOps][kMaxParams];
  __shared__ uint8_t s_fired[kMaxOps];
  if (threadIdx.x == 0) sample_image(a, i, s_prm, s_fired);
  __syncthreads();
  const int v = threadIdx.x;
  for (int s = 0; s < a.n_luts; ++s) {
    for (int c = 0; c < 3; ++c) {
      int x = v;
      for (int k = a.lut_k0[s]; k < a.lut_k1[s]; ++k)
        if (s_fired[k]) x = lut_entry(a.ops[k].kind, s_prm[k], c, x);
      a.luts[((size_t)i * a.n_luts + s) * 768 + c * 256 + v] = (uint8_t)x;
    }
  }
  if (a.norm_slot >= 0 && blockIdx.x == 0) {  // per plan; every launch writes the same values
    const alb_op& o = a.ops[a.norm_slot];
    for (int c = 0; c < 3; ++c)
      a.norm_lut[c * 256 + v] =
          (float)__ddiv_rn(__dsub_rn(__ddiv_rn((double)v, 255.0), o.mean[c]), o.std[c]);
  }
}

// no LUT to build: one thread per image (a 256-thread CTA per image would
// leave 255 threads idle and cost a block-scheduling wave per ~1200 images)
__global__ void __launch_bounds__(128) k_prep_lite(PrepArgs a) {
  const int i = a.img0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.img0 + a.n) sample_image(a, i, nullptr, nullptr);
}

void launch_prep(const PrepArgs& a, cudaStream_t s) {
  if (a.n <= 0) return;
  if (a.n_luts == 0 && a.norm_slot < 0) k_prep_lite<<<(a.n + 127) / 128, 128, 0, s>>>(a);
  else k_prep<<<a.n, 256, 0, s>>>(a);
}

}  // namespace alb
