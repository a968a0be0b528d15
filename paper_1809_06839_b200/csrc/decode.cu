// decode.cu -- GPU input front-end (PAPER.md:56-57:
// GPUs idle while the CPU prepares batches): a batch of JPEG bitstreams in host
// memory decoded by nvJPEG straight into a ragged u8 RGB layout, i.e. the
// input of alb_apply, on the caller's stream.  The B200's hardware JPEG
// engines are used when nvJPEG's hardware backend accepts the batch, else its
// CUDA backend.  nvJPEG is a library (like cuBLAS); it is loaded with dlopen
// on first use, so the augmentation library itself has no link dependency on
// it.  Host code only.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvjpeg.h>

#include <string>
#include <type_traits>
#include <vector>

#include "config.h"

using namespace alb;

namespace {

struct NvJpeg {
  void* so = nullptr;
  decltype(&nvjpegCreateEx) create_ex = nullptr;
  decltype(&nvjpegDestroy) destroy = nullptr;
  decltype(&nvjpegJpegStateCreate) state_create = nullptr;
  decltype(&nvjpegJpegStateDestroy) state_destroy = nullptr;
  decltype(&nvjpegGetImageInfo) image_info = nullptr;
  decltype(&nvjpegDecodeBatchedInitialize) batched_init = nullptr;
  decltype(&nvjpegDecodeBatched) batched = nullptr;
};

// resolve nvJPEG once per process; empty string on success
const std::string& load_nvjpeg(NvJpeg& f) {
  static NvJpeg g;
  static std::string err = [] {
    const char* names[] = {"libnvjpeg.so.12", "libnvjpeg.so"};
    for (const char* n : names)
      if ((g.so = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
    if (!g.so) return std::string("nvJPEG not found (dlopen libnvjpeg.so.12)");
    bool ok = true;
    auto sym = [&](auto& fp, const char* name) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(g.so, name));
      ok = ok && fp != nullptr;
    };
    sym(g.create_ex, "nvjpegCreateEx");
    sym(g.destroy, "nvjpegDestroy");
    sym(g.state_create, "nvjpegJpegStateCreate");
    sym(g.state_destroy, "nvjpegJpegStateDestroy");
    sym(g.image_info, "nvjpegGetImageInfo");
    sym(g.batched_init, "nvjpegDecodeBatchedInitialize");
    sym(g.batched, "nvjpegDecodeBatched");
    return ok ? std::string() : std::string("nvJPEG: missing symbols");
  }();
  f = g;
  return err;
}

}  // namespace

struct alb_decoder {
  NvJpeg f;
  nvjpegHandle_t h = nullptr;
  nvjpegJpegState_t st = nullptr;
  int backend = 0;     // 1 = hardware engines
  int batch = -1;      // batch size the state is initialised for
  ~alb_decoder() {
    if (st) f.state_destroy(st);
    if (h) f.destroy(h);
  }
};

extern "C" {

alb_status alb_decoder_create(int32_t prefer_hardware, alb_decoder** out) {
  if (!out) return set_error(ALB_E_INVALID_ARG, "null out");
  auto* d = new alb_decoder;
  const std::string& e = load_nvjpeg(d->f);
  if (!e.empty()) { delete d; return set_error(ALB_E_UNSUPPORTED, e); }
  // hardware JPEG engines, else GPU-assisted Huffman decoding (the default
  // backend decodes Huffman on one CPU thread), else the default backend
  nvjpegStatus_t s = NVJPEG_STATUS_IMPLEMENTATION_NOT_SUPPORTED;
  if (prefer_hardware) {
    s = d->f.create_ex(NVJPEG_BACKEND_HARDWARE, nullptr, nullptr, 0, &d->h);
    d->backend = s == NVJPEG_STATUS_SUCCESS ? 1 : 0;
  }
  if (s != NVJPEG_STATUS_SUCCESS) {
    s = d->f.create_ex(NVJPEG_BACKEND_GPU_HYBRID, nullptr, nullptr, 0, &d->h);
    d->backend = s == NVJPEG_STATUS_SUCCESS ? 2 : 0;
  }
  if (s != NVJPEG_STATUS_SUCCESS) s = d->f.create_ex(NVJPEG_BACKEND_DEFAULT, nullptr, nullptr, 0, &d->h);
  if (s != NVJPEG_STATUS_SUCCESS) { d->h = nullptr; delete d; return set_error(ALB_E_CUDA, "nvjpegCreateEx failed"); }
  if (d->f.state_create(d->h, &d->st) != NVJPEG_STATUS_SUCCESS) {
    d->st = nullptr;
    delete d;
    return set_error(ALB_E_CUDA, "nvjpegJpegStateCreate failed");
  }
  *out = d;
  return ALB_OK;
}

void alb_decoder_destroy(alb_decoder* d) { delete d; }

int32_t alb_decoder_backend(const alb_decoder* d) { return d ? d->backend : -1; }

alb_status alb_jpeg_info(alb_decoder* d, const uint8_t* data, size_t length, int32_t* height, int32_t* width) {
  if (!d || !data || !height || !width) return set_error(ALB_E_INVALID_ARG, "null argument");
  int nc = 0;
  nvjpegChromaSubsampling_t sub;
  int w[NVJPEG_MAX_COMPONENT], h[NVJPEG_MAX_COMPONENT];
  if (d->f.image_info(d->h, data, length, &nc, &sub, w, h) != NVJPEG_STATUS_SUCCESS || nc < 1)
    return set_error(ALB_E_INVALID_ARG, "not a decodable JPEG bitstream");
  *height = h[0];
  *width = w[0];
  return ALB_OK;
}

alb_status alb_decode_jpeg(alb_decoder* d, const uint8_t* const* data, const size_t* lengths, int32_t n,
                           const alb_layout* out, uint8_t* dev_out, void* stream) {
  if (!d || !out || n < 0 || (n > 0 && (!data || !lengths || !dev_out))) return set_error(ALB_E_INVALID_ARG, "null argument");
  const std::vector<alb_image_desc>& desc = layout_desc(out);
  if ((int)desc.size() != n) return set_error(ALB_E_SHAPE, "layout holds a different number of images");
  if (layout_channels(out) != 3) return set_error(ALB_E_UNSUPPORTED, "decode writes 3-channel RGB layouts");
  if (n == 0) return ALB_OK;
  std::vector<nvjpegImage_t> dst(n);
  for (int i = 0; i < n; ++i) {
    int32_t h, w;
    alb_status s = alb_jpeg_info(d, data[i], lengths[i], &h, &w);
    if (s) return set_error(s, "image " + std::to_string(i) + ": not a decodable JPEG bitstream");
    if (h != desc[i].height || w != desc[i].width)
      return set_error(ALB_E_SHAPE, "image " + std::to_string(i) + ": JPEG dims differ from the layout");
    dst[i] = nvjpegImage_t{};
    dst[i].channel[0] = dev_out + desc[i].offset;
    dst[i].pitch[0] = (size_t)desc[i].pitch;
  }
  if (d->batch != n) {
    if (d->f.batched_init(d->h, d->st, n, 1, NVJPEG_OUTPUT_RGBI) != NVJPEG_STATUS_SUCCESS)
      return set_error(ALB_E_CUDA, "nvjpegDecodeBatchedInitialize failed");
    d->batch = n;
  }
  const nvjpegStatus_t s = d->f.batched(d->h, d->st, data, lengths, dst.data(), (cudaStream_t)stream);
  if (s != NVJPEG_STATUS_SUCCESS) {
    d->batch = -1;  // re-initialise next time
    return set_error(s == NVJPEG_STATUS_JPEG_NOT_SUPPORTED || s == NVJPEG_STATUS_IMPLEMENTATION_NOT_SUPPORTED ? ALB_E_UNSUPPORTED
                                                                                                  : ALB_E_CUDA,
                     "nvjpegDecodeBatched failed (status " + std::to_string((int)s) + ")");
  }
  return ALB_OK;
}

}  // extern "C"
