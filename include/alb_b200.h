/*
 * alb_b200.h -- C ABI of the B200-native augmentation hot path of
 * arXiv 1809.06839 ("Albumentations: fast and flexible image augmentations").
 *
 * The problem statement (BASELINE.json north_star): apply a
 * pipeline of transforms T with parameters p to a batch of images, with masks
 * and bounding boxes co-transformed (Fig. 2), each transform
 * applied iff its gate draw u < p.  The transforms are the ones
 * the paper's benchmark times (Table 1) plus the configs of
 * BASELINE.json; their exact definitions are DESIGN.md O0-O14.
 *
 * Every pixel of every step runs in hand-written sm_100a CUDA kernels.  There
 * is no CPU fallback: without a CUDA device the calls return ALB_E_CUDA.
 *
 * Conventions
 *  - Pixel / mask / box buffers passed to alb_apply are DEVICE pointers owned
 *    by the caller.  The library owns only its opaque handles (pipeline,
 *    layout, plan), the small device tables a plan uploads at creation and a
 *    small pool of side streams per (device, host thread) for label / box
 *    work, which alb_plan_create creates for its thread.  alb_apply allocates
 *    no memory; it creates the pool only when called with a masked / boxed
 *    plan from a thread other than the one that created the plan.
 *  - Images are HWC uint8, RGB, row-major, x = column, y = row, origin top
 *    left.  A batch is ragged: image i lives at
 *    base + desc[i].offset with desc[i].pitch >= width*channels bytes per row.
 *    Every 32-byte-aligned block that contains a byte of an image must be
 *    readable (the kernels read whole aligned 16- / 32-byte blocks; allocate
 *    batches with >= 32 bytes of slack at both ends or on 32-byte aligned
 *    sizes; torch caching-allocator blocks satisfy this).
 *  - Boxes are normalized xyxy float32, [n][max_boxes][4],
 *    with a per-image count; labels int32 [n][max_boxes] (optional).
 *  - Randomness: parameters of (image i, op slot k) are a pure function of
 *    (seed, first_image_index + i, k) through Philox4x32-10 (O1), so
 *    results do not depend on how a batch is split across calls or GPUs.
 *  - Validation is atomic: every check happens on the host
 *    before anything is enqueued; on error nothing is launched.
 *  - alb_apply is asynchronous on `stream` (a cudaStream_t passed as void*)
 *    and never synchronises.  Device faults surface at the caller's sync.
 *  - Handles are immutable after creation and may be shared across threads
 *    and streams; each concurrent alb_apply needs its own
 *    workspace.
 */
#ifndef ALB_B200_H
#define ALB_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ALB_OK = 0,
  ALB_E_INVALID_ARG = -1,  /* null/overlapping buffers, window larger than image */
  ALB_E_UNKNOWN_OP = -2,   /* kind outside alb_kind */
  ALB_E_RANGE = -3,        /* p outside [0,1], lo > hi, beta < 0, g <= 0, scale <= 0 */
  ALB_E_SHAPE = -4,        /* mask dims != image dims, output layout dims mismatch */
  ALB_E_UNSUPPORTED = -5,  /* 1-channel image to an RGB-only op, too many ops */
  ALB_E_ALIGN = -6,        /* descriptor offsets/pitches violate the layout rules */
  ALB_E_CUDA = -7,         /* CUDA error (no device, launch failure) */
  ALB_E_WORKSPACE = -8     /* workspace missing or smaller than alb_plan_workspace_size */
} alb_status;

/* Transform kinds.  Numbering is part of the contract. */
typedef enum {
  ALB_HFLIP = 0,                 /* PAPER.md:125; O2                             */
  ALB_VFLIP = 1,                 /* PAPER.md:126; O2                             */
  ALB_ROTATE = 2,                /* PAPER.md:127; O7  params: theta (deg)        */
  ALB_SHIFT_SCALE_ROTATE = 3,    /* PAPER.md:128; O7  params: dx, dy, scale, theta */
  ALB_RANDOM_CROP = 4,           /* PAPER.md:123; O3  out_w x out_h              */
  ALB_PAD_TO_SIZE = 5,           /* PAPER.md:124; O4  out_w x out_h, fill        */
  ALB_RESIZE = 6,                /* PAPER.md:86 "scaling"; O5                    */
  ALB_RANDOM_SIZED_CROP = 7,     /* PAPER.md:76; O6   side in [min_side,max_side] -> out */
  ALB_BRIGHTNESS = 8,            /* PAPER.md:129; O8  params: beta               */
  ALB_CONTRAST = 9,              /* PAPER.md:64;  O8  params: c                  */
  ALB_BRIGHTNESS_CONTRAST = 10,  /* BASELINE cfg2/4; O8/R12 params: beta, c      */
  ALB_GAMMA = 11,                /* PAPER.md:132; O8  params: g                  */
  ALB_SHIFT_RGB = 12,            /* PAPER.md:131; O8  params: dr, dg, db         */
  ALB_SHIFT_HSV = 13,            /* PAPER.md:130; O9  params: dh (deg), ds, dv   */
  ALB_GRAYSCALE = 14,            /* PAPER.md:133; O10                            */
  ALB_EQUALIZE = 15,             /* BASELINE cfg2; O11/R15                       */
  ALB_NORMALIZE = 16,            /* BASELINE cfg4; O12/R16 -> fp32 NCHW, last op */
  ALB_CROP = 17,                 /* PAPER.md:37 "cropping"; O3 fixed window      */
  ALB_ROT90 = 18,                /* PAPER.md:87; SPEC.md:193-201 k quarter turns
                                    (counter-clockwise as displayed), k uniform in
                                    the integer range [lo[0], hi[0]] within 0..3   */
  ALB_D4 = 19,                   /* PAPER.md:87 "dihedral group"
                                    element e uniform in [lo[0], hi[0]] within 0..7:
                                    e < 4 -> rot90(e), else hflip(rot90(e - 4))   */
  ALB_GRID_DISTORTION = 20,      /* PAPER.md Fig. 4 "grid distortion"; SPEC.md:329-337;
                                    reading R31: num_steps cells per axis, cell
                                    lengths proportional to factors 1 + U(lo[0], hi[0])
                                    (-1 < lo <= hi < 1), span preserved; bilinear or
                                    nearest remap (border unused: maps stay inside);
                                    masks nearest; boxes rejected (ALB_E_UNSUPPORTED) */
  ALB_ELASTIC = 21,              /* PAPER.md:102 "elastic transform"; SPEC.md:338-346;
                                    reading R32: alpha = lo[0] (>= 0), sigma = lo[1]
                                    (0 < sigma <= 16), both fixed (lo == hi); raw
                                    U(-1,1) planes from Philox, fp64 Gaussian blur
                                    (radius ceil(3 sigma), reflect-101), remap at
                                    (x + dx, y + dy) with interp / border / fill;
                                    masks nearest; boxes rejected                  */
  ALB_NUM_KINDS = 22
} alb_kind;

typedef enum { ALB_INTERP_NEAREST = 0, ALB_INTERP_BILINEAR = 1 } alb_interp;
typedef enum { ALB_BORDER_CONSTANT = 0, ALB_BORDER_REFLECT_101 = 1 } alb_border;

/* One transform (SPEC.md:470-474 TransformSpec).  Continuous parameter j is
 * drawn as lo[j] + (hi[j]-lo[j])*u_j (O1); lo == hi fixes it.
 * Shape-changing kinds (RandomCrop, Crop, PadToSize, Resize, RandomSizedCrop)
 * require p == 1 (reading R17) so batch output shapes are static.  Rot90 / D4
 * transpose the shape for odd elements: on a non-square image every outcome
 * (including an unfired gate) must have the same parity, else the plan fails
 * with ALB_E_UNSUPPORTED (reading R30). */
typedef struct {
  int32_t kind;
  double p;
  double lo[4], hi[4];
  int32_t out_w, out_h;          /* RandomCrop / Crop / PadToSize / Resize / RSC */
  int32_t min_side, max_side;    /* RandomSizedCrop side range in pixels (R6)    */
  int32_t crop_x, crop_y;        /* Crop window origin                           */
  int32_t interp, border;        /* alb_interp, alb_border                       */
  uint8_t fill[3], mask_fill;    /* constant-border / pad fill                   */
  double mean[3], std[3];        /* Normalize                                    */
  int32_t num_steps;             /* GridDistortion cells per axis, 1..ALB_GRID_MAX_STEPS */
  int32_t reserved;              /* unused                                       */
} alb_op;

#define ALB_GRID_MAX_STEPS 32

/* Geometry of image i of a ragged batch (bytes). */
typedef struct {
  int64_t offset;
  int32_t height, width, pitch;
  int32_t reserved;
} alb_image_desc;

typedef struct alb_pipeline alb_pipeline;
typedef struct alb_layout alb_layout;
typedef struct alb_plan alb_plan;

#define ALB_MAX_OPS 16
#define ALB_MAX_PARAMS 8

/* Validate and copy an op list ("params validate ... before any
 * pixel work").  *out owned by the caller; free with alb_pipeline_destroy.
 * Errors: ALB_E_UNKNOWN_OP, ALB_E_RANGE, ALB_E_UNSUPPORTED (n_ops > ALB_MAX_OPS). */
alb_status alb_pipeline_create(const alb_op* ops, int32_t n_ops, alb_pipeline** out);
void alb_pipeline_destroy(alb_pipeline* p);

/* Output dims for an in_h x in_w input.  ALB_E_INVALID_ARG when a window
 * op does not fit. */
alb_status alb_output_shape(const alb_pipeline* p, int32_t in_h, int32_t in_w,
                            int32_t* out_h, int32_t* out_w);

/* Describe a ragged batch: desc is a HOST array [n], copied (and uploaded to
 * the device) by the call.  channels is 3 for images, 1 for masks.
 * Errors: ALB_E_SHAPE (h, w < 1), ALB_E_ALIGN (pitch < w*channels, negative
 * offset), ALB_E_CUDA. */
alb_status alb_layout_create(const alb_image_desc* desc, int32_t n, int32_t channels,
                             alb_layout** out);
void alb_layout_destroy(alb_layout* l);

/* Bind a pipeline to batch layouts and build the launch plan (kernel
 * selection / fusion, work tables).  This is SURVEY.md §8(b)'s alb_batch +
 * alb_workspace_size split in two: the geometry of a batch (alb_layout) and
 * the fusion decisions depend only on the op list and the image sizes, so
 * they are computed and uploaded once here instead of on every apply; the
 * per-step inputs (seed, image index, buffers) stay in alb_apply.  The
 * transforms are applied in list order with every
 * op's u8 rounding kept, masks nearest
 * and boxes clipped once at the end (readings R18, R19).  `out` is NULL iff the pipeline ends in
 * Normalize (the output is then fp32 NCHW [n][3][oh][ow], all images must map
 * to one output size).  mask_in/mask_out both NULL or both set (1-channel,
 * same dims as the images).  max_boxes > 0 enables box co-transform with the
 * given min_visibility (reading R19).  Errors: ALB_E_SHAPE (layout dims differ
 * from alb_output_shape), ALB_E_UNSUPPORTED, ALB_E_INVALID_ARG. */
alb_status alb_plan_create(const alb_pipeline* p, const alb_layout* in, const alb_layout* out,
                           const alb_layout* mask_in, const alb_layout* mask_out,
                           int32_t max_boxes, float min_visibility, alb_plan** plan);
void alb_plan_destroy(alb_plan* plan);
alb_status alb_plan_workspace_size(const alb_plan* plan, size_t* bytes);
/* Number of kernel launches one alb_apply of this plan enqueues (the
 * single-pass Equalize counted as one launch: it is taken when the buffers
 * are 16-byte co-aligned, as device allocations are; otherwise Equalize runs
 * as histogram + LUT + LUT-pass kernels, two more). */
int32_t alb_plan_num_launches(const alb_plan* plan);

/* Apply the plan to one batch (device pointers): SPEC.md:482-490 apply(p,
 * bundle, seed) for a whole batch -- "apply transform T with parameters p to
 * image/mask/bboxes" (BASELINE.json north_star; Fig. 2).  The
 * seed is an argument here rather than a pipeline field (SURVEY.md §8(b)
 * puts it in alb_pipeline_create): the pipeline and plan stay immutable while
 * a training loop advances the seed per step (SPEC.md:485 seed_override).
 * Image i of the batch uses global index first_image_index + i (< 2^32);
 * its gate and parameters are draws (seed, first_image_index + i, slot) of
 * Philox4x32-10, so the output does not depend on how a
 * batch is split across calls or GPUs (SPEC.md:502 determinism).  Boxes: boxes_in [n][max_boxes][4],
 * labels_in [n][max_boxes] or NULL, count_in [n]; outputs likewise (kept
 * boxes compacted stably to the front, count_out = kept count).
 * Asynchronous on `stream`: it enqueues kernels (and, for Equalize, a
 * memset of its histogram workspace) and nothing else -- no host
 * synchronisation, allocation or copy -- so it can be captured into a CUDA
 * graph and replayed (seed and pointers are baked into the graph).  Label
 * (mask) and box work may run on a library-owned side stream (one of a
 * pool of 4 per device and host thread, always the same one for a given
 * `stream`, so applies on different caller streams overlap their label
 * work too), forked from `stream` by an event after the
 * work already enqueued there and joined back into `stream` before the call
 * returns, so `stream` ordering holds as if everything ran on it; if that
 * stream could not be created, the label / box work runs on `stream`.
 * Errors: ALB_E_INVALID_ARG (null required pointer, in/out overlap),
 * ALB_E_WORKSPACE, ALB_E_CUDA (launch failure). */
alb_status alb_apply(const alb_plan* plan, uint64_t seed, uint64_t first_image_index,
                     const uint8_t* img_in, uint8_t* img_out, float* out_nchw,
                     const uint8_t* mask_in, uint8_t* mask_out,
                     const float* boxes_in, const int32_t* labels_in, const int32_t* count_in,
                     float* boxes_out, int32_t* labels_out, int32_t* count_out,
                     void* workspace, size_t workspace_bytes, void* stream);

/* End-to-end variant with HOST buffers (pinned for async copies): copies the
 * input batch host->device into dev_in, applies, copies the output
 * device->host (no sync).  in_bytes / out_bytes are the flat buffer sizes of
 * the batch buffers (layout offsets index into them).  When the layouts'
 * images lie in increasing, disjoint byte ranges the batch runs as up to 16
 * image chunks: H2D copies on a plan-owned stream, the kernels of each chunk
 * on `stream`, D2H copies on a second plan-owned stream, chained by events, so
 * copies in both directions overlap the kernels; the work is ordered after
 * everything earlier on `stream` and everything later on `stream` sees the
 * host output complete.  One alb_apply_host per plan at a time.  Masks and
 * boxes are not carried by this entry point (ALB_E_UNSUPPORTED). */
alb_status alb_apply_host(const alb_plan* plan, uint64_t seed, uint64_t first_image_index,
                          const uint8_t* host_in, size_t in_bytes, uint8_t* dev_in,
                          void* host_out, size_t out_bytes, void* dev_out,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Parameters the device sampler draws (bit-identical to what alb_apply uses):
 * SPEC.md:485 "draw gate = uniform_f64() (always drawn, even when p=1) ...
 * then draw that transform's parameters in its documented order", with the
 * counter-based layout of SURVEY.md §8(c) O1.  params_out HOST
 * [n][n_ops][ALB_MAX_PARAMS], fired_out HOST [n][n_ops]; in_hw HOST [n][2]
 * (height, width) of each input image -- RandomCrop / RandomSizedCrop draw
 * their windows from the size each slot sees, which is why
 * this call takes sizes and a seed beyond §8(b)'s signature.  Runs the same
 * device sampler as alb_apply, then copies back; synchronous.  Errors:
 * ALB_E_INVALID_ARG (null pointers, n < 0, a window larger than the image),
 * ALB_E_SHAPE (dims < 1), ALB_E_CUDA. */
alb_status alb_sample_params(const alb_pipeline* p, uint64_t seed, uint64_t first_image_index,
                             const int32_t* in_hw, int32_t n, double* params_out,
                             uint8_t* fired_out);

/* Thread-local message for the last non-OK status of this thread. */
/* Pipeline configs: UTF-8 JSON
 *   {"seed": <optional u64>, "transforms": [{"name": "<kind>", "p": <number>,
 *                                            "params": {...}}, ...]}
 * with the kind names of alb_kind's comments (HorizontalFlip, ..., ElasticTransform)
 * and per-kind params (range params take a number = fixed value or [lo, hi]):
 *   Rotate {angle, interpolation?, border?, fill?, mask_fill?}
 *   ShiftScaleRotate {shift_x, shift_y, scale, angle, interpolation?, border?, fill?, mask_fill?}
 *   RandomCrop {width, height}   Crop {x, y, width, height}   PadToSize {width, height, fill?, mask_fill?}
 *   Resize {width, height, interpolation?}   RandomSizedCrop {min_side, max_side, width, height, interpolation?}
 *   Brightness {beta}  Contrast {c}  BrightnessContrast {beta, c}  Gamma {g}
 *   ShiftRGB {dr, dg, db}  ShiftHSV {dh, ds, dv}  Normalize {mean[3], std[3]}
 *   Rotate90 {k}  D4 {element}  GridDistortion {num_steps, distort_limit (d = [-d, d]), interpolation?}
 *   ElasticTransform {alpha, sigma (numbers), interpolation?, border?, fill?, mask_fill?}
 *   HorizontalFlip, VerticalFlip, Grayscale, Equalize: {}
 * interpolation "nearest" | "bilinear" (default), border "constant" (default) |
 * "reflect_101", fill [r, g, b] (default 0), mask_fill (default 0).  "p" is
 * mandatory.  from_json: text NUL-terminated; *out as alb_pipeline_create;
 * seed / has_seed (may be NULL) receive the optional seed.  Errors:
 * ALB_E_INVALID_ARG (syntax, type, unknown field, missing required param --
 * alb_last_error names it), ALB_E_UNKNOWN_OP (message lists the valid names),
 * ALB_E_RANGE / ALB_E_UNSUPPORTED as alb_pipeline_create.
 * to_json: every param of each kind written explicitly, numbers round-trip
 * exact; *len = bytes excluding the NUL; buf may be NULL to query the size,
 * else cap must be >= *len + 1 (ALB_E_INVALID_ARG).  seed NULL = no seed field. */
alb_status alb_pipeline_from_json(const char* text, alb_pipeline** out, uint64_t* seed, int32_t* has_seed);
alb_status alb_pipeline_to_json(const alb_pipeline* p, const uint64_t* seed, char* buf, size_t cap, size_t* len);

/* GPU input front-end ("GPUs idle
 * while the CPU prepares batches"): JPEG bitstreams in HOST memory decoded by
 * nvJPEG (a library, loaded with dlopen on first use) into a ragged RGB u8
 * layout on the device -- the input of alb_apply.
 * alb_decoder_create: prefer_hardware != 0 asks for nvJPEG's hardware backend
 *   (the GPU's JPEG engines), falling back to its CUDA backend.  Errors:
 *   ALB_E_UNSUPPORTED (nvJPEG missing), ALB_E_CUDA.  One decoder per stream /
 *   thread at a time.
 * alb_decoder_backend: 1 = hardware engines, 2 = GPU-assisted Huffman, 0 = default backend.
 * alb_jpeg_info: dims of a bitstream (host parse) for building the layout.
 * alb_decode_jpeg: data[i] / lengths[i] host bitstreams (caller-owned, valid
 *   until the stream reaches this point), out a 3-channel layout whose image i
 *   has the bitstream's dims (ALB_E_SHAPE otherwise), dev_out its device base.
 *   Asynchronous on `stream`; ALB_E_UNSUPPORTED for bitstreams nvJPEG rejects. */
typedef struct alb_decoder alb_decoder;
alb_status alb_decoder_create(int32_t prefer_hardware, alb_decoder** out);
void alb_decoder_destroy(alb_decoder* d);
int32_t alb_decoder_backend(const alb_decoder* d);
alb_status alb_jpeg_info(alb_decoder* d, const uint8_t* data, size_t length, int32_t* height, int32_t* width);
alb_status alb_decode_jpeg(alb_decoder* d, const uint8_t* const* data, const size_t* lengths, int32_t n,
                           const alb_layout* out, uint8_t* dev_out, void* stream);

const char* alb_last_error(void);
int32_t alb_version(void);

#ifdef __cplusplus
}
#endif
#endif
