// resample.cu -- K5 Resize / RandomSizedCrop (O5/O6) with fused
// post-ops: exact flips/crops on the output coordinates, the pointwise stage
// chain (HSV / LUT / gray) and Normalize-to-fp32-NCHW output (K9, cfg4).
//
// Half-pixel bilinear: x_s = (x_d + 0.5) * ww / nw - 0.5, clamped to the
// window [0, ww-1] (replicate border at the WINDOW edge, R9).  Column and row
// tables (x0, fx, nearest) are computed in fp64 in the definition's operation
// order, so the coordinates equal the oracle's bit for bit; the blend runs in
// fp32.  Masks: nearest, round_half_up(x_s).
//
// Work unit = (image, band of `unit_rows` output rows); persistent grid over
// contiguous unit ranges; the column table is rebuilt only when the image
// changes.  Per band, the window rows it needs are staged in shared memory as
// RGBx words (16-byte loads + byte permutes); each lane then computes one
// output pixel per (row, 32-pixel segment) from 4 shared-memory taps and the
// warp writes the segment with shuffled 4-byte stores.
#include "stages.cuh"

namespace alb {

constexpr int kRsThreads = 256;
constexpr int kRsMaxCols = 2048;
constexpr int kRsMaxBand = 64;

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

struct ColEnt {
  int x0;      // tap 0 column (window frame); tap 1 = min(x0+1, ww-1)
  float fx;
  int xn;      // nearest column
  int x1;
};

__global__ void __launch_bounds__(kRsThreads) k_resample(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  StageCtx x;
  init_stages(a, x);
  ColEnt* col = reinterpret_cast<ColEnt*>(sm + x.n_lut * kLutWords);
  int* row_y0 = reinterpret_cast<int*>(col + kRsMaxCols);
  float* row_fy = reinterpret_cast<float*>(row_y0 + kRsMaxBand);
  int* row_yn = reinterpret_cast<int*>(row_fy + kRsMaxBand);
  int* s_geom = row_yn + kRsMaxBand;
  uint32_t* stage = reinterpret_cast<uint32_t*>(s_geom + 8);
  const bool nearest = a.interp == ALB_INTERP_NEAREST;
  const bool has_mask = a.mdst != nullptr;
  const int R = a.unit_rows;

  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  RsGeom g{};
  Map1 m{};
  int Wo = 0, Ho = 0;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    const int img = unit.x;
    __syncthreads();
    if (img != cur_img) {
      load_stages(a, img, sm, x, kRsThreads);
      g = rs_geom(a, img);
      Wo = a.normalize ? a.out_w : a.ddesc[img].width;
      Ho = a.normalize ? a.out_h : a.ddesc[img].height;
      m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, Wo, Ho);
      for (int xo = threadIdx.x; xo < Wo; xo += kRsThreads) {
        const int xr = m.ax * xo + m.bx;
        const double s = rs_coord(xr, g.ww, g.nw);
        const double f = floor(s);
        ColEnt e;
        e.x0 = (int)f;
        e.x1 = min(e.x0 + 1, g.ww - 1);
        e.fx = (float)__dsub_rn(s, f);
        e.xn = (int)floor(__dadd_rn(s, 0.5));
        col[xo] = e;
      }
      cur_img = img;
    }
    const int y0 = unit.y * R, y1 = min(Ho, y0 + R);
    if (threadIdx.x < y1 - y0) {
      const int yr = m.ay * (y0 + threadIdx.x) + m.by;
      const double s = rs_coord(yr, g.wh, g.nh);
      const double f = floor(s);
      row_y0[threadIdx.x] = (int)f;
      row_fy[threadIdx.x] = (float)__dsub_rn(s, f);
      row_yn[threadIdx.x] = (int)floor(__dadd_rn(s, 0.5));
    }
    __syncthreads();
    // rows of the window this band needs (monotone in y up to the flip)
    int ra = row_y0[0], rb = row_y0[y1 - y0 - 1];
    const int sy_lo = min(ra, rb);
    const int sy_hi = min(max(ra, rb) + 1, g.wh - 1);
    const int nrows = sy_hi - sy_lo + 1;
    const int S = g.ww;
    const bool staged = (long long)nrows * S <= a.unit_size;
    const alb_image_desc sd = a.sdesc[img];
    const uint8_t* wbase = a.src + sd.offset + (size_t)g.wy0 * sd.pitch + (size_t)g.wx0 * 3;
    if (staged) {
      const int per_row = (g.ww + 15) / 16;
      for (int it = threadIdx.x; it < nrows * per_row; it += kRsThreads) {
        const int r = it / per_row, c16 = (it % per_row) * 16;
        const uint8_t* srow = a.src + sd.offset + (size_t)(g.wy0 + sy_lo + r) * sd.pitch;
        uint32_t w[12];
        load_window<12>(srow + (size_t)(g.wx0 + c16) * 3, srow, srow + (size_t)sd.width * 3, w);
        uint32_t* d = stage + r * S + c16;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c16 + i < g.ww) d[i] = rgbx_of(w, i);
      }
      __syncthreads();
    }
    const int nseg = (Wo + 31) / 32;
    for (int rs = warp; rs < (y1 - y0) * nseg; rs += kRsThreads / 32) {
      const int rr = rs / nseg, seg = rs % nseg;
      const int yo = y0 + rr;
      const int xo = seg * 32 + lane;
      const int nvalid = min(32, Wo - seg * 32);
      const bool act = lane < nvalid;
      const ColEnt ce = col[act ? xo : 0];
      uint32_t r, gg, b;
      if (nearest) {
        const int yn = row_yn[rr];
        const uint32_t t = staged ? stage[(yn - sy_lo) * S + ce.xn]
                                  : (wbase[(size_t)yn * sd.pitch + 3 * ce.xn] |
                                     (wbase[(size_t)yn * sd.pitch + 3 * ce.xn + 1] << 8) |
                                     (wbase[(size_t)yn * sd.pitch + 3 * ce.xn + 2] << 16));
        r = t & 0xff; gg = (t >> 8) & 0xff; b = (t >> 16) & 0xff;
      } else {
        const int ry0 = row_y0[rr];
        const int ry1 = min(ry0 + 1, g.wh - 1);
        const float fy = row_fy[rr];
        uint32_t t00, t10, t01, t11;
        if (staged) {
          const uint32_t* p0 = stage + (ry0 - sy_lo) * S;
          const uint32_t* p1 = stage + (ry1 - sy_lo) * S;
          t00 = p0[ce.x0]; t10 = p0[ce.x1]; t01 = p1[ce.x0]; t11 = p1[ce.x1];
        } else {
          const uint8_t* q0 = wbase + (size_t)ry0 * sd.pitch;
          const uint8_t* q1 = wbase + (size_t)ry1 * sd.pitch;
          t00 = q0[3 * ce.x0] | (q0[3 * ce.x0 + 1] << 8) | (q0[3 * ce.x0 + 2] << 16);
          t10 = q0[3 * ce.x1] | (q0[3 * ce.x1 + 1] << 8) | (q0[3 * ce.x1 + 2] << 16);
          t01 = q1[3 * ce.x0] | (q1[3 * ce.x0 + 1] << 8) | (q1[3 * ce.x0 + 2] << 16);
          t11 = q1[3 * ce.x1] | (q1[3 * ce.x1 + 1] << 8) | (q1[3 * ce.x1 + 2] << 16);
        }
        uint32_t ch[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float p00 = (float)((t00 >> (8 * c)) & 0xff), p10 = (float)((t10 >> (8 * c)) & 0xff);
          const float p01 = (float)((t01 >> (8 * c)) & 0xff), p11 = (float)((t11 >> (8 * c)) & 0xff);
          const float h0 = fmaf(ce.fx, p10 - p00, p00);
          const float h1 = fmaf(ce.fx, p11 - p01, p01);
          const float v = fmaf(fy, h1 - h0, h0);
          ch[c] = (uint32_t)(v + 0.5f);
        }
        r = ch[0]; gg = ch[1]; b = ch[2];
      }
      apply_stages(x, sm, lane, r, gg, b);
      if (a.normalize) {
        if (act) {
          const size_t plane = (size_t)Ho * Wo;
          float* o = a.nchw + (size_t)img * 3 * plane + (size_t)yo * Wo + xo;
          const float* nl = a.tab.norm_lut;
          __stcs(o, nl[r]);
          __stcs(o + plane, nl[256 + gg]);
          __stcs(o + 2 * plane, nl[512 + b]);
        }
      } else {
        const alb_image_desc dd = a.ddesc[img];
        uint8_t* drow = a.dst + dd.offset + (size_t)yo * dd.pitch + (size_t)seg * 32 * 3;
        warp_store_rgb(drow, nvalid, r | (gg << 8) | (b << 16), lane);
      }
      if (has_mask && act) {
        const alb_image_desc msd = a.msdesc[img];
        const alb_image_desc mdd = a.mddesc[img];
        const uint8_t* mw = a.msrc + msd.offset + (size_t)g.wy0 * msd.pitch + g.wx0;
        a.mdst[mdd.offset + (size_t)yo * mdd.pitch + xo] = mw[(size_t)row_yn[rr] * msd.pitch + ce.xn];
      }
    }
  }
}

size_t resample_smem(const StepArgs& a) {
  return (size_t)count_lut_stages(a) * kLutWords * 4 + sizeof(ColEnt) * kRsMaxCols +
         kRsMaxBand * 12 + 32 + (size_t)a.unit_size * 4;
}

void launch_resample(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const size_t smem = resample_smem(a);
  cudaFuncSetAttribute(k_resample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1, sms = 148, dev = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_resample, kRsThreads, smem);
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(a.n_units, sms * std::max(occ, 1));
  k_resample<<<grid, kRsThreads, smem, s>>>(a);
}

}  // namespace alb
