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
// RGBx words (16-byte loads + byte permutes).  Each warp owns output rows:
// lane = column, 4 shared-memory taps per pixel, RGB bytes into a per-warp
// shared row buffer, then the warp writes the row with aligned 16-byte stores.
#include <algorithm>

#include "stages.cuh"

namespace alb {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsMaxCols = 2048;
constexpr int kRsMaxBand = 64;
constexpr int kRsChunk = 512;  // output columns per row-buffer flush

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
  uint16_t x0, xn;  // tap-0 and nearest columns (window frame)
  float fx;
};

struct RsState {
  RsGeom g;
  Map1 m;
  int Wo, Ho;
  int sy_lo, nrows, staged, pad;
};

// kGeneric = false: bilinear, u8 output -- the uniform mode branches compile
// away (a predicated-off Normalize path would otherwise issue per pixel)
template <int kOne, bool kGeneric>
__global__ void __launch_bounds__(kRsThreads, 3) k_resample(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  StageCtx x;
  init_stages(a, x);
  ColEnt* col = reinterpret_cast<ColEnt*>(sm + x.n_lut * kLutWords);
  int* row_y0 = reinterpret_cast<int*>(col + kRsMaxCols);
  float* row_fy = reinterpret_cast<float*>(row_y0 + kRsMaxBand);
  int* row_yn = reinterpret_cast<int*>(row_fy + kRsMaxBand);
  RsState* st = reinterpret_cast<RsState*>(row_yn + kRsMaxBand);
  uint8_t* rowbuf = reinterpret_cast<uint8_t*>(st + 1) + warp * (kRsChunk * 3 + 32);
  uint32_t* stage = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(st + 1) +
                                                kRsWarps * (kRsChunk * 3 + 32));
  const bool nearest = kGeneric && a.interp == ALB_INTERP_NEAREST;
  const bool has_mask = a.mdst != nullptr;
  const bool normalize = kGeneric && a.normalize;
  const int R = a.unit_rows;

  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    const int img = unit.x;
    __syncthreads();
    if (img != cur_img) {
      load_stages(a, img, sm, x, kRsThreads);
      const RsGeom g = rs_geom(a, img);
      const int Wo = a.normalize ? a.out_w : a.ddesc[img].width;
      const int Ho = a.normalize ? a.out_h : a.ddesc[img].height;
      const Map1 m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, Wo, Ho);
      for (int xo = threadIdx.x; xo < Wo; xo += kRsThreads) {
        const double s = rs_coord(m.ax * xo + m.bx, g.ww, g.nw);
        const double f = floor(s);
        ColEnt e;
        e.x0 = (uint16_t)(int)f;
        e.xn = (uint16_t)(int)floor(__dadd_rn(s, 0.5));
        e.fx = (float)__dsub_rn(s, f);
        col[xo] = e;
      }
      if (threadIdx.x == 0) {
        st->g = g; st->m = m; st->Wo = Wo; st->Ho = Ho;
      }
      cur_img = img;
      __syncthreads();
    }
    const RsGeom g = st->g;
    const Map1 m = st->m;
    const int Wo = st->Wo, Ho = st->Ho;
    const int y0 = unit.y * R, y1 = min(Ho, y0 + R);
    if (threadIdx.x < y1 - y0) {
      const double s = rs_coord(m.ay * (y0 + threadIdx.x) + m.by, g.wh, g.nh);
      const double f = floor(s);
      row_y0[threadIdx.x] = (int)f;
      row_fy[threadIdx.x] = (float)__dsub_rn(s, f);
      row_yn[threadIdx.x] = (int)floor(__dadd_rn(s, 0.5));
    }
    __syncthreads();
    // window rows this band needs (the row map is monotone)
    const int ra = row_y0[0], rb = row_y0[y1 - y0 - 1];
    const int sy_lo = min(ra, rb);
    const int nrows = min(max(ra, rb) + 1, g.wh - 1) - sy_lo + 1;
    const int S = g.ww;
    const bool staged = (long long)nrows * S <= a.unit_size;
    const alb_image_desc sd = a.sdesc[img];
    const uint8_t* wbase = a.src + sd.offset + (size_t)g.wy0 * sd.pitch + (size_t)g.wx0 * 3;
    if (staged) {
      const int per_row = (g.ww + 15) >> 4;
      const uint32_t magic = 0xffffffffu / (uint32_t)per_row + 1u;
      for (int it = threadIdx.x; it < nrows * per_row; it += kRsThreads) {
        const int r = per_row == 1 ? it : (int)__umulhi((uint32_t)it, magic);
        const int c16 = (it - r * per_row) << 4;
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
    uint8_t* dbase = nullptr;
    int dpitch = 0;
    if (!normalize) {
      const alb_image_desc dd = a.ddesc[img];
      dbase = a.dst + dd.offset;
      dpitch = dd.pitch;
    }
    const size_t plane = (size_t)Ho * Wo;
    float* nbase = normalize ? a.nchw + (size_t)img * 3 * plane : nullptr;
    const float* nl = a.tab.norm_lut;
    for (int rr = warp; rr < y1 - y0; rr += kRsWarps) {
      const int yo = y0 + rr;
      const int ry0 = row_y0[rr];
      const int ry1 = min(ry0 + 1, g.wh - 1);
      const float fy = row_fy[rr];
      const uint32_t* p0 = stage + (ry0 - sy_lo) * S;
      const uint32_t* p1 = stage + (ry1 - sy_lo) * S;
      const uint8_t* q0 = wbase + (size_t)ry0 * sd.pitch;
      const uint8_t* q1 = wbase + (size_t)ry1 * sd.pitch;
      for (int cx0 = 0; cx0 < Wo; cx0 += kRsChunk) {
        const int cw = min(kRsChunk, Wo - cx0);
        for (int c = lane; c < cw; c += 32) {
          const int xo = cx0 + c;
          const ColEnt ce = col[xo];
          uint32_t r, gg, b;
          if (nearest) {
            const int yn = row_yn[rr];
            uint32_t t;
            if (staged) {
              t = stage[(yn - sy_lo) * S + ce.xn];
            } else {
              const uint8_t* q = wbase + (size_t)yn * sd.pitch + 3 * ce.xn;
              t = q[0] | (q[1] << 8) | (q[2] << 16);
            }
            r = t & 0xff; gg = (t >> 8) & 0xff; b = (t >> 16) & 0xff;
          } else {
            const int x0 = ce.x0, x1 = min(x0 + 1, g.ww - 1);
            uint32_t t00, t10, t01, t11;
            if (staged) {
              t00 = p0[x0]; t10 = p0[x1]; t01 = p1[x0]; t11 = p1[x1];
            } else {
              t00 = q0[3 * x0] | (q0[3 * x0 + 1] << 8) | (q0[3 * x0 + 2] << 16);
              t10 = q0[3 * x1] | (q0[3 * x1 + 1] << 8) | (q0[3 * x1 + 2] << 16);
              t01 = q1[3 * x0] | (q1[3 * x0 + 1] << 8) | (q1[3 * x0 + 2] << 16);
              t11 = q1[3 * x1] | (q1[3 * x1 + 1] << 8) | (q1[3 * x1 + 2] << 16);
            }
            const uint32_t px = bilerp_rgbx(t00, t10, t01, t11, ce.fx, fy);
            r = px & 0xff; gg = (px >> 8) & 0xff; b = (px >> 16) & 0xff;
          }
          apply_stages_t<kOne>(x, sm, lane, r, gg, b);
          if (normalize) {
            float* o = nbase + (size_t)yo * Wo + xo;
            __stcs(o, nl[r]);
            __stcs(o + plane, nl[256 + gg]);
            __stcs(o + 2 * plane, nl[512 + b]);
          } else {
            rowbuf[3 * c] = (uint8_t)r;
            rowbuf[3 * c + 1] = (uint8_t)gg;
            rowbuf[3 * c + 2] = (uint8_t)b;
          }
        }
        if (!normalize) {
          __syncwarp();
          warp_copy_row(dbase + (size_t)yo * dpitch + (size_t)cx0 * 3, rowbuf, 3 * cw, lane);
          __syncwarp();
        }
      }
      if (has_mask) {
        const alb_image_desc msd = a.msdesc[img];
        const alb_image_desc mdd = a.mddesc[img];
        const uint8_t* mrow = a.msrc + msd.offset + (size_t)(g.wy0 + row_yn[rr]) * msd.pitch + g.wx0;
        uint8_t* mo = a.mdst + mdd.offset + (size_t)yo * mdd.pitch;
        for (int xo = lane; xo < Wo; xo += 32) mo[xo] = mrow[col[xo].xn];
      }
    }
  }
}

static size_t resample_smem(const StepArgs& a) {
  return (size_t)count_lut_stages(a) * kLutWords * 4 + sizeof(ColEnt) * kRsMaxCols +
         kRsMaxBand * 12 + sizeof(RsState) + kRsWarps * (kRsChunk * 3 + 32) +
         (size_t)a.unit_size * 4;
}

template <int kOne, bool kGeneric>
static void launch_resample_v(const StepArgs& a, size_t smem, cudaStream_t s) {
  const int grid = persistent_grid((const void*)k_resample<kOne, kGeneric>, kRsThreads, smem, a.n_units);
  k_resample<kOne, kGeneric><<<grid, kRsThreads, smem, s>>>(a);
}

template <int kOne>
static void launch_resample_t(const StepArgs& a, size_t smem, cudaStream_t s) {
  if (a.normalize || a.interp == ALB_INTERP_NEAREST) launch_resample_v<kOne, true>(a, smem, s);
  else launch_resample_v<kOne, false>(a, smem, s);
}

void launch_resample(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const size_t smem = resample_smem(a);
  const int mode = stage_mode(a);
  ALB_DISPATCH_STAGES(mode, launch_resample_t, a, smem, s)
}

}  // namespace alb
