// resample.cu -- K5 Resize / RandomSizedCrop (O5/O6) with fused
// post-ops: exact flips/crops on the output coordinates, the pointwise stage
// chain (HSV / LUT / gray) and Normalize-to-fp32-NCHW output (K9, cfg4).
//
// Half-pixel bilinear: x_s = (x_d + 0.5) * ww / nw - 0.5, clamped to the
// window [0, ww-1] (replicate border at the WINDOW edge, R9).  The column and
// row tables (x0, x1, fx) are computed once per CTA in fp64 exactly as the
// definition orders the operations, so coordinates match the oracle to the
// last bit; the blend runs in fp32.  Masks: nearest, round_half_up(x_s).
//
// Work unit = (image, band of output rows).  The source window's rows are
// staged into shared memory as RGBx words (one 32-bit word per pixel) with
// 16-byte vector loads, then every output pixel reads its 4 taps from shared
// memory.  Each thread produces one aligned 16-pixel block.
#include "stages.cuh"

namespace alb {

constexpr int kRsThreads = 256;
constexpr int kRsMaxCols = 2048;   // output width limit of the table path
constexpr int kRsBand = 16;        // output rows per unit

struct RsGeom {
  int wx0, wy0, ww, wh;  // source window
  int nw, nh;            // resize output dims
};

__device__ __forceinline__ RsGeom rs_geom(const StepArgs& a, int img) {
  const alb_op& o = a.ops[a.slot0];
  RsGeom g;
  g.nw = o.out_w;
  g.nh = o.out_h;
  if (o.kind == ALB_RANDOM_SIZED_CROP) {
    const double* q = prm_of(a.tab, img, a.slot0);
    g.ww = g.wh = (int)q[0];
    g.wx0 = (int)q[1];
    g.wy0 = (int)q[2];
  } else {
    g.wx0 = g.wy0 = 0;
    g.ww = dim_w(a.tab, img, a.slot0);
    g.wh = dim_h(a.tab, img, a.slot0);
  }
  return g;
}

// source coordinate of output index d along one axis (fp64, definition order)
__device__ __forceinline__ double rs_coord(int d, int n_src, int n_dst) {
  double s = __dsub_rn(__ddiv_rn(__dmul_rn(__dadd_rn((double)d, 0.5), (double)n_src), (double)n_dst), 0.5);
  if (s < 0.0) s = 0.0;
  if (s > (double)(n_src - 1)) s = (double)(n_src - 1);
  return s;
}

__global__ void __launch_bounds__(kRsThreads) k_resample(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  const int lane = threadIdx.x & 31;
  const alb_image_desc sd = a.sdesc[img];
  const int Wo = a.normalize ? a.out_w : a.ddesc[img].width;
  const int Ho = a.normalize ? a.out_h : a.ddesc[img].height;
  const RsGeom g = rs_geom(a, img);
  const Map1 m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, Wo, Ho);
  const int y0 = unit.y * kRsBand;
  const int y1 = min(Ho, y0 + kRsBand);

  StageCtx x;
  load_stages(a, img, sm, x, kRsThreads);
  uint32_t* smx = sm + x.n_lut * kLutWords;
  int* col_x0 = reinterpret_cast<int*>(smx);            // [Wo] source column of tap 0 (window frame)
  float* col_fx = reinterpret_cast<float*>(col_x0 + kRsMaxCols);
  int* col_xn = reinterpret_cast<int*>(col_fx + kRsMaxCols);  // nearest (masks)
  int* row_y0 = col_xn + kRsMaxCols;                    // [band]
  float* row_fy = reinterpret_cast<float*>(row_y0 + kRsBand);
  int* row_yn = reinterpret_cast<int*>(row_fy + kRsBand);
  uint32_t* stage = reinterpret_cast<uint32_t*>(row_yn + kRsBand);  // staged source rows (RGBx)

  for (int xo = threadIdx.x; xo < Wo; xo += kRsThreads) {
    const int xr = m.ax * xo + m.bx;  // resize-output column
    const double s = rs_coord(xr, g.ww, g.nw);
    const double f = floor(s);
    col_x0[xo] = (int)f;
    col_fx[xo] = (float)__dsub_rn(s, f);
    col_xn[xo] = (int)floor(__dadd_rn(s, 0.5));
  }
  // source rows needed by this band
  int sy_lo = 1 << 30, sy_hi = -1;
  for (int yy = y0; yy < y1; ++yy) {
    const int yr = m.ay * yy + m.by;
    const double s = rs_coord(yr, g.wh, g.nh);
    const int f = (int)floor(s);
    sy_lo = min(sy_lo, f);
    sy_hi = max(sy_hi, min(f + 1, g.wh - 1));
    if (threadIdx.x == 0) {
      row_y0[yy - y0] = f;
      row_fy[yy - y0] = (float)__dsub_rn(s, floor(s));
      row_yn[yy - y0] = (int)floor(__dadd_rn(s, 0.5));
    }
  }
  const int nrows = sy_hi - sy_lo + 1;
  const int stride = g.ww;  // words per staged row
  const bool staged = a.unit_size > 0 && nrows * stride <= a.unit_size;
  if (staged) {
    // stage window rows [sy_lo, sy_hi] x [wx0, wx0+ww) as RGBx words; 16 px per item
    const int per_row = (g.ww + 15) / 16;
    for (int it = threadIdx.x; it < nrows * per_row; it += kRsThreads) {
      const int r = it / per_row, c16 = (it % per_row) * 16;
      const uint8_t* srow = a.src + sd.offset + (size_t)(g.wy0 + sy_lo + r) * sd.pitch;
      uint32_t w[12];
      load_window<12>(srow + (size_t)(g.wx0 + c16) * 3, srow, srow + (size_t)sd.width * 3, w);
      uint32_t* d = stage + r * stride + c16;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (c16 + i < g.ww)
          d[i] = byte_of(w, 3 * i) | (byte_of(w, 3 * i + 1) << 8) | (byte_of(w, 3 * i + 2) << 16);
      }
    }
  }
  __syncthreads();

  const uint8_t* wbase = a.src + sd.offset + (size_t)g.wy0 * sd.pitch + (size_t)g.wx0 * 3;
  const int nbmax = 2 + Wo / 16;
  const int items = (y1 - y0) * nbmax;
  for (int it = threadIdx.x; it < items; it += kRsThreads) {
    const int yy = y0 + it / nbmax;
    const int k = it % nbmax - 1;
    int xb;
    uint8_t* drow = nullptr;
    if (a.normalize) {
      xb = 16 * k;
    } else {
      const alb_image_desc dd = a.ddesc[img];
      drow = a.dst + dd.offset + (size_t)yy * dd.pitch;
      xb = first_aligned_px_offset<3>((uintptr_t)drow) / 3 + 16 * k;
    }
    if (xb + 16 <= 0 || xb >= Wo) continue;
    const int ry0 = row_y0[yy - y0];
    const int ry1 = min(ry0 + 1, g.wh - 1);
    const float fy = row_fy[yy - y0];
    uint32_t px[48];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int xo = min(max(xb + i, 0), Wo - 1);
      const int cx0 = col_x0[xo];
      const int cx1 = min(cx0 + 1, g.ww - 1);
      const float fx = col_fx[xo];
      uint32_t t00, t10, t01, t11;
      if (staged) {
        const uint32_t* r0 = stage + (ry0 - sy_lo) * stride;
        const uint32_t* r1 = stage + (ry1 - sy_lo) * stride;
        t00 = r0[cx0]; t10 = r0[cx1]; t01 = r1[cx0]; t11 = r1[cx1];
      } else {
        const uint8_t* p0 = wbase + (size_t)ry0 * sd.pitch;
        const uint8_t* p1 = wbase + (size_t)ry1 * sd.pitch;
        t00 = p0[3 * cx0] | (p0[3 * cx0 + 1] << 8) | (p0[3 * cx0 + 2] << 16);
        t10 = p0[3 * cx1] | (p0[3 * cx1 + 1] << 8) | (p0[3 * cx1 + 2] << 16);
        t01 = p1[3 * cx0] | (p1[3 * cx0 + 1] << 8) | (p1[3 * cx0 + 2] << 16);
        t11 = p1[3 * cx1] | (p1[3 * cx1 + 1] << 8) | (p1[3 * cx1 + 2] << 16);
      }
      uint32_t ch[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float p00 = (float)((t00 >> (8 * c)) & 0xff), p10 = (float)((t10 >> (8 * c)) & 0xff);
        const float p01 = (float)((t01 >> (8 * c)) & 0xff), p11 = (float)((t11 >> (8 * c)) & 0xff);
        const float h0 = (1.f - fx) * p00 + fx * p10;
        const float h1 = (1.f - fx) * p01 + fx * p11;
        const float v = (1.f - fy) * h0 + fy * h1;
        ch[c] = (uint32_t)min(255, (int)floorf(v + 0.5f));
      }
      apply_stages(a, x, sm, lane, ch[0], ch[1], ch[2]);
      px[3 * i] = ch[0]; px[3 * i + 1] = ch[1]; px[3 * i + 2] = ch[2];
    }
    if (a.normalize) {
      store_nchw(a, img, yy, xb, px, Wo, Ho);
    } else {
      uint32_t w[12];
#pragma unroll
      for (int q = 0; q < 12; ++q)
        w[q] = px[4 * q] | (px[4 * q + 1] << 8) | (px[4 * q + 2] << 16) | (px[4 * q + 3] << 24);
      store_block<3>(drow, xb, Wo, w);
    }
  }

  // mask (nearest), byte-wise
  if (a.mdst) {
    const alb_image_desc msd = a.msdesc[img];
    const alb_image_desc mdd = a.mddesc[img];
    const uint8_t* mw = a.msrc + msd.offset + (size_t)g.wy0 * msd.pitch + g.wx0;
    for (int it = threadIdx.x; it < (y1 - y0) * Wo; it += kRsThreads) {
      const int yy = y0 + it / Wo, xo = it % Wo;
      a.mdst[mdd.offset + (size_t)yy * mdd.pitch + xo] =
          mw[(size_t)row_yn[yy - y0] * msd.pitch + col_xn[xo]];
    }
  }
}

size_t resample_smem(const StepArgs& a) {
  return (size_t)count_lut_stages(a) * kLutWords * 4 + (size_t)kRsMaxCols * 12 + kRsBand * 12 +
         (size_t)a.unit_size * 4;
}

void launch_resample(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const size_t smem = resample_smem(a);
  cudaFuncSetAttribute(k_resample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_resample<<<a.n_units, kRsThreads, smem, s>>>(a);
}

}  // namespace alb
