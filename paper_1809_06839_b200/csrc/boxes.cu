// boxes.cu -- K11 bounding-box co-transform (O13, readings R18/R19).
// One warp per image.  Boxes are carried in pixel-edge coordinates of the
// current frame, unclipped, through every fired geometric op of the pipeline
// (flips, crops, pad, resize/RSC, Rotate/SSR via the 4 corners in the
// pixel-centre frame and their envelope); at the end they are clipped to the
// output image, kept iff non-empty and clipped area >= min_visibility *
// unclipped area, and compacted stably with a ballot prefix.  fp64 throughout
// with explicit round-to-nearest intrinsics (no contraction).
#include "kernels.cuh"

namespace alb {

__device__ void box_through_op(const alb_op& o, const double* q, int hin, int win, double& X0,
                               double& Y0, double& X1, double& Y1) {
  switch (o.kind) {
    case ALB_HFLIP: {
      const double a = __dsub_rn((double)win, X1), b = __dsub_rn((double)win, X0);
      X0 = a; X1 = b;
      break;
    }
    case ALB_VFLIP: {
      const double a = __dsub_rn((double)hin, Y1), b = __dsub_rn((double)hin, Y0);
      Y0 = a; Y1 = b;
      break;
    }
    case ALB_CROP: case ALB_RANDOM_CROP:
      X0 = __dsub_rn(X0, q[0]); X1 = __dsub_rn(X1, q[0]);
      Y0 = __dsub_rn(Y0, q[1]); Y1 = __dsub_rn(Y1, q[1]);
      break;
    case ALB_PAD_TO_SIZE: {
      const double left = (double)((o.out_w - win) / 2), top = (double)((o.out_h - hin) / 2);
      X0 = __dadd_rn(X0, left); X1 = __dadd_rn(X1, left);
      Y0 = __dadd_rn(Y0, top); Y1 = __dadd_rn(Y1, top);
      break;
    }
    case ALB_RESIZE: case ALB_RANDOM_SIZED_CROP: {
      double wx0 = 0, wy0 = 0, ww = win, wh = hin;
      if (o.kind == ALB_RANDOM_SIZED_CROP) { ww = wh = q[0]; wx0 = q[1]; wy0 = q[2]; }
      X0 = __ddiv_rn(__dmul_rn(__dsub_rn(X0, wx0), (double)o.out_w), ww);
      X1 = __ddiv_rn(__dmul_rn(__dsub_rn(X1, wx0), (double)o.out_w), ww);
      Y0 = __ddiv_rn(__dmul_rn(__dsub_rn(Y0, wy0), (double)o.out_h), wh);
      Y1 = __ddiv_rn(__dmul_rn(__dsub_rn(Y1, wy0), (double)o.out_h), wh);
      break;
    }
    case ALB_ROTATE: case ALB_SHIFT_SCALE_ROTATE: {
      double dx = 0, dy = 0, s = 1, th;
      if (o.kind == ALB_SHIFT_SCALE_ROTATE) { dx = q[0]; dy = q[1]; s = q[2]; th = q[3]; } else { th = q[0]; }
      const double rad = __ddiv_rn(__dmul_rn(th, 3.141592653589793), 180.0);
      const double cs = cos(rad), sn = sin(rad);
      const double cx = __ddiv_rn(__dsub_rn((double)win, 1.0), 2.0);
      const double cy = __ddiv_rn(__dsub_rn((double)hin, 1.0), 2.0);
      const double tx = __dmul_rn(dx, (double)win), ty = __dmul_rn(dy, (double)hin);
      double lx = 0, hx = 0, ly = 0, hy = 0;
      for (int k = 0; k < 4; ++k) {
        const double X = (k & 1) ? X1 : X0, Y = (k & 2) ? Y1 : Y0;
        const double xc = __dsub_rn(X, 0.5) , yc = __dsub_rn(Y, 0.5);
        const double ux = __dsub_rn(xc, cx), uy = __dsub_rn(yc, cy);
        const double xp = __dadd_rn(__dadd_rn(cx, __dmul_rn(s, __dadd_rn(__dmul_rn(cs, ux), __dmul_rn(sn, uy)))), tx);
        const double yp = __dadd_rn(__dadd_rn(cy, __dmul_rn(s, __dadd_rn(__dmul_rn(-sn, ux), __dmul_rn(cs, uy)))), ty);
        const double Xp = __dadd_rn(xp, 0.5), Yp = __dadd_rn(yp, 0.5);
        if (k == 0 || Xp < lx) lx = Xp;
        if (k == 0 || Xp > hx) hx = Xp;
        if (k == 0 || Yp < ly) ly = Yp;
        if (k == 0 || Yp > hy) hy = Yp;
      }
      X0 = lx; X1 = hx; Y0 = ly; Y1 = hy;
      break;
    }
    case ALB_ROT90: case ALB_D4: {  // (x, y) -> (y, 1 - x) per quarter turn
      const int e = (int)q[0];
      double w = win;
      for (int t = 0; t < (e & 3); ++t) {  // pixel-edge frame: (X, Y) -> (Y, w - X)
        const double nx0 = Y0, nx1 = Y1, ny0 = __dsub_rn(w, X1), ny1 = __dsub_rn(w, X0);
        w = (t & 1) ? (double)win : (double)hin;  // width of the frame after this turn
        X0 = nx0; X1 = nx1; Y0 = ny0; Y1 = ny1;
      }
      if (e >= 4) {  // then hflip in the rotated frame
        const double a = __dsub_rn(w, X1), b = __dsub_rn(w, X0);
        X0 = a; X1 = b;
      }
      break;
    }
    default: break;
  }
}

__global__ void __launch_bounds__(128) k_boxes(BoxArgs a) {
  const int img = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (img >= a.n) return;
  const int cnt = min(a.count_in[img], a.max_boxes);
  const int H0 = dim_h(a.tab, img, 0), W0 = dim_w(a.tab, img, 0);
  const int n_ops = a.tab.n_ops;
  const int Hf = dim_h(a.tab, img, n_ops), Wf = dim_w(a.tab, img, n_ops);
  int base = 0;
  for (int j0 = 0; j0 < cnt; j0 += 32) {
    const int j = j0 + lane;
    bool keep = false;
    float o[4] = {0, 0, 0, 0};
    int lab = 0;
    if (j < cnt) {
      const float* b = a.boxes_in + ((size_t)img * a.max_boxes + j) * 4;
      double X0 = __dmul_rn((double)b[0], (double)W0), Y0 = __dmul_rn((double)b[1], (double)H0);
      double X1 = __dmul_rn((double)b[2], (double)W0), Y1 = __dmul_rn((double)b[3], (double)H0);
      for (int k = 0; k < n_ops; ++k) {
        if (!fired_of(a.tab, img, k)) continue;
        box_through_op(a.ops[k], prm_of(a.tab, img, k), dim_h(a.tab, img, k), dim_w(a.tab, img, k),
                       X0, Y0, X1, Y1);
      }
      const double area = __dmul_rn(__dsub_rn(X1, X0), __dsub_rn(Y1, Y0));
      const double cx0 = X0 < 0.0 ? 0.0 : X0, cy0 = Y0 < 0.0 ? 0.0 : Y0;
      const double cx1 = X1 > (double)Wf ? (double)Wf : X1;
      const double cy1 = Y1 > (double)Hf ? (double)Hf : Y1;
      if (cx1 > cx0 && cy1 > cy0) {
        const double carea = __dmul_rn(__dsub_rn(cx1, cx0), __dsub_rn(cy1, cy0));
        keep = carea >= __dmul_rn((double)a.min_visibility, area);
      }
      o[0] = (float)__ddiv_rn(cx0, (double)Wf);
      o[1] = (float)__ddiv_rn(cy0, (double)Hf);
      o[2] = (float)__ddiv_rn(cx1, (double)Wf);
      o[3] = (float)__ddiv_rn(cy1, (double)Hf);
      lab = a.labels_in ? a.labels_in[(size_t)img * a.max_boxes + j] : 0;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int pos = base + __popc(bal & ((1u << lane) - 1u));
      float* d = a.boxes_out + ((size_t)img * a.max_boxes + pos) * 4;
      d[0] = o[0]; d[1] = o[1]; d[2] = o[2]; d[3] = o[3];
      if (a.labels_out) a.labels_out[(size_t)img * a.max_boxes + pos] = lab;
    }
    base += __popc(bal);
  }
  if (lane == 0) a.count_out[img] = base;
}

void launch_boxes(const BoxArgs& a, cudaStream_t s) {
  if (a.n > 0) k_boxes<<<(a.n + 3) / 4, 128, 0, s>>>(a);
}

}  // namespace alb
