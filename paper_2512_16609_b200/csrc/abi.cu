// C ABI of libdehaze_b200.so (see include/dehaze_b200.h).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdarg>
#include <string>

#include "../../include/dehaze_b200.h"
#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace {
thread_local std::string g_err;
}  // namespace

namespace dhz {
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("DHZ_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

int abi_fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
int abi_cuda_fail(cudaError_t e, const char* where) {
  return abi_fail(DHZ_E_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}
}  // namespace dhz

namespace {

#define fail dhz::abi_fail
inline int cuda_fail(cudaError_t e, const char* where) { return dhz::abi_cuda_fail(e, where); }

constexpr int64_t kAlign = 256;
constexpr int kMaxFrames = 65535;  // frames ride grid.y / grid.z

// Stage events: inside a CUDA-graph capture they become event-record nodes
// (external records), so a replayed graph still timestamps every stage.
void record_stage_event(void* const* events, int i, cudaStream_t st) {
  if (!events || !events[i]) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(reinterpret_cast<cudaEvent_t>(events[i]), st, cudaEventRecordExternal);
  else
    cudaEventRecord(reinterpret_cast<cudaEvent_t>(events[i]), st);
}
int64_t align_up(int64_t v, int64_t a = kAlign) { return (v + a - 1) / a * a; }

struct Layout {
  // [0, zero_end) is cleared at the start of every call
  int64_t frame_max, sel, unit_max, row_hist, frame_hist, hist256, full_list, zero_end;
  int64_t row_info, sel_idx, lut, bal, dark, tmap, total;
  int64_t dark_fs;
};

Layout make_layout(int n, int H, int W, const dhz_params* p) {
  Layout L{};
  const int64_t npx = (int64_t)H * W;
  L.dark_fs = align_up(npx, 16);
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = align_up(o + bytes);
    return at;
  };
  const int64_t nb = (H + dhz::kBandH - 1) / dhz::kBandH, nu = (W + dhz::kUnitW - 1) / dhz::kUnitW;
  L.frame_max = take(4LL * n);
  L.sel = take((int64_t)sizeof(dhz::FrameSel) * n);
  L.unit_max = take(4LL * n * nb * nu);
  L.row_hist = take(4LL * dhz::kWin * n * H);
  L.frame_hist = take(4LL * dhz::kWin * n);
  L.hist256 = take(4LL * 256 * n);
  L.full_list = take(4LL * (n + 1));
  L.zero_end = o;
  L.row_info = take(16LL * n * H);
  L.sel_idx = take(4LL * n * std::max<int64_t>(1, p->top_k));
  if (p->mode == 1) {  // image mode: guided-filter scratch instead of the LUT
    L.lut = L.bal = -1;
    L.tmap = take((int64_t)dhz::guided_ws_bytes(n, H, W, p->guided_radius, p->balance != 0));
  } else {
    L.lut = take((int64_t)dhz::kLutFrame * n);
    L.bal = p->balance ? take((int64_t)dhz::balance_ws_bytes(n)) : -1;
    L.tmap = -1;
  }
  L.dark = take(L.dark_fs * n);
  L.total = o;
  return L;
}

int check_params(int n, int H, int W, const dhz_params* p) {
  if (!p) return fail(DHZ_E_INVALID, "params is NULL");
  if (n < 0) return fail(DHZ_E_INVALID, "n_frames must be >= 0, got %d", n);
  if (n > kMaxFrames) return fail(DHZ_E_INVALID, "n_frames %d above %d per call (grid limit): split the batch", n, kMaxFrames);
  if (H < 1 || W < 1) return fail(DHZ_E_INVALID, "empty frame %dx%d", W, H);
  const int64_t npx = (int64_t)H * W;
  if (npx > 0xFFFFFFF0LL) return fail(DHZ_E_INVALID, "frame too large (%lld px)", (long long)npx);
  if (p->top_k < 1 || p->top_k > npx)
    return fail(DHZ_E_INVALID, "top_k must lie in [1, %lld], got %lld", (long long)npx, (long long)p->top_k);
  if (p->patch_radius < 1) return fail(DHZ_E_INVALID, "patch_radius must be >= 1");
  if (!p->thresholds) return fail(DHZ_E_INVALID, "thresholds table is NULL");
  if (p->mode != 0 && p->mode != 1) return fail(DHZ_E_INVALID, "mode must be 0 or 1");
  return DHZ_OK;
}

}  // namespace

extern "C" {

const char* dhz_last_error(void) { return g_err.c_str(); }

int dhz_abi_version(void) { return DHZ_ABI_VERSION; }

int dhz_device_count(void) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n < 1) {
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    return fail(DHZ_E_CUDA, "no CUDA device visible");
  }
  return n;
}

size_t dhz_frames_u8_workspace(int n, int height, int width, const dhz_params* p) {
  if (check_params(std::max(n, 0), height, width, p) != DHZ_OK) return 0;
  return (size_t)make_layout(n, height, width, p).total;
}

int dhz_frames_u8_layout(int n, int height, int width, const dhz_params* p, int64_t* off) {
  int rc = check_params(n, height, width, p);
  if (rc) return rc;
  if (!off) return fail(DHZ_E_INVALID, "offsets is NULL");
  const Layout L = make_layout(n, height, width, p);
  off[0] = L.dark;
  off[1] = L.dark_fs;
  off[2] = L.sel_idx;
  off[3] = L.tmap;
  off[4] = L.total;
  return DHZ_OK;
}

}  // extern "C"

namespace {

// Shared argument checks of the native-size entry points.
int frames_check(const uint8_t* in, int64_t in_fs, int n, int H, int W, const dhz_params* p, const void* out,
                 int64_t out_fs, const double* airlight, void* ws, size_t ws_bytes, const Layout& L) {
  if (!in || !out || !airlight) return fail(DHZ_E_INVALID, "NULL array argument");
  const int64_t npx = (int64_t)H * W;
  if (in_fs < 3 * npx || out_fs < 3 * npx) return fail(DHZ_E_INVALID, "frame stride smaller than a frame");
  if (!ws || (int64_t)ws_bytes < L.total)
    return fail(DHZ_E_WORKSPACE, "workspace too small: need %lld bytes, got %zu", (long long)L.total, ws_bytes);
  if (p->mode == 1 && (p->guided_radius < 1 || p->guided_radius > dhz::kGuidedMaxRadius))
    return fail(DHZ_E_UNSUPPORTED, "guided_radius %d outside [1, %d] of the fused guided filter",
                p->guided_radius, dhz::kGuidedMaxRadius);
  if (dhz::dark_u8_max_smem(p->patch_radius) > 200 * 1024)
    return fail(DHZ_E_UNSUPPORTED, "patch_radius %d too large for the tiled erosion", p->patch_radius);
  return DHZ_OK;
}

// K1 dark channel + K2-K4 top-K select and airlight (events [0]..[2]).
int frames_airlight(const uint8_t* in, int64_t in_fs, int n, int H, int W, const dhz_params* p, double* airlight,
                    uint8_t* base, const Layout& L, cudaStream_t st, void* const* events) {
  auto mark = [&](int i) { record_stage_event(events, i, st); };
  mark(0);
  cudaError_t e = cudaMemsetAsync(base, 0, (size_t)L.zero_end, st);  // maxima, select state, histograms
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  const int64_t npx = (int64_t)H * W;
  uint8_t* dark = base + L.dark;
  uint32_t* fmax = reinterpret_cast<uint32_t*>(base + L.frame_max);
  uint32_t* umax = reinterpret_cast<uint32_t*>(base + L.unit_max);
  e = dhz::dark_u8(in, in_fs, n, H, W, p->patch_radius, dark, L.dark_fs, fmax, umax, st);
  if (e != cudaSuccess) return cuda_fail(e, "dark_u8");
  mark(1);
  dhz::SelectWs sw{};
  sw.sel = reinterpret_cast<dhz::FrameSel*>(base + L.sel);
  sw.frame_max = fmax;
  sw.unit_max = umax;
  sw.row_hist = reinterpret_cast<uint32_t*>(base + L.row_hist);
  sw.frame_hist = reinterpret_cast<uint32_t*>(base + L.frame_hist);
  sw.hist256 = reinterpret_cast<uint32_t*>(base + L.hist256);
  sw.full_list = reinterpret_cast<uint32_t*>(base + L.full_list);
  sw.row_info = reinterpret_cast<uint32_t*>(base + L.row_info);
  sw.sel_idx = reinterpret_cast<uint32_t*>(base + L.sel_idx);
  sw.H = H;
  sw.W = W;
  e = dhz::select_u8(dark, L.dark_fs, in, in_fs, n, npx, p->top_k, p->alpha, sw, airlight, st);
  if (e != cudaSuccess) return cuda_fail(e, "select_u8");
  mark(2);
  return DHZ_OK;
}

// Transmission (+ guided filter) + recovery + postprocess + output from a given
// airlight (events [3], [4]).
int frames_recover(const uint8_t* in, int64_t in_fs, int n, int H, int W, const dhz_params* p,
                   const double* airlight, uint8_t* out, int64_t out_fs, uint8_t* base, const Layout& L,
                   cudaStream_t st, void* const* events) {
  auto mark = [&](int i) { record_stage_event(events, i, st); };
  cudaError_t e;
  if (p->mode == 1) {  // guided filter + recovery (+ gray-world) fused; event 3 == event 4
    e = dhz::guided_recover_u8(in, in_fs, n, H, W, p->guided_radius, p->guided_eps, airlight, p->omega, p->t_min,
                               p->thresholds, p->gamma, p->balance != 0, out, out_fs, base + L.tmap, st);
    if (e != cudaSuccess) return cuda_fail(e, "guided_recover_u8");
    mark(3);
    mark(4);
    return DHZ_OK;
  }
  uint8_t* lut = base + L.lut;
  if (p->balance)
    e = dhz::build_lut_balanced_u8(in, in_fs, n, H, W, airlight, p->omega, p->t_min, p->gamma, lut, base + L.bal,
                                   st);
  else
    e = dhz::build_lut_u8(n, airlight, p->omega, p->t_min, p->thresholds, p->gamma, lut, st);
  if (e != cudaSuccess) return cuda_fail(e, "build_lut_u8");
  mark(3);
  e = dhz::recover_lut_u8(in, in_fs, n, H, W, lut, out, out_fs, st);
  if (e != cudaSuccess) return cuda_fail(e, "recover_lut_u8");
  mark(4);
  return DHZ_OK;
}

}  // namespace

extern "C" {

int dhz_frames_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, const dhz_params* p, uint8_t* out,
                  int64_t out_fs, double* airlight, void* ws, size_t ws_bytes, void* stream,
                  void* const* events) {
  int rc = check_params(n, H, W, p);
  if (rc) return rc;
  if (n == 0) return DHZ_OK;
  const Layout L = make_layout(n, H, W, p);
  if ((rc = frames_check(in, in_fs, n, H, W, p, out, out_fs, airlight, ws, ws_bytes, L))) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  if ((rc = frames_airlight(in, in_fs, n, H, W, p, airlight, base, L, st, events))) return rc;
  return frames_recover(in, in_fs, n, H, W, p, airlight, out, out_fs, base, L, st, events);
}

int dhz_frames_u8_airlight(const uint8_t* in, int64_t in_fs, int n, int H, int W, const dhz_params* p,
                           double* airlight, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_params(n, H, W, p);
  if (rc) return rc;
  if (n == 0) return DHZ_OK;
  const Layout L = make_layout(n, H, W, p);
  if ((rc = frames_check(in, in_fs, n, H, W, p, airlight, 3LL * H * W, airlight, ws, ws_bytes, L))) return rc;
  return frames_airlight(in, in_fs, n, H, W, p, airlight, static_cast<uint8_t*>(ws), L,
                         reinterpret_cast<cudaStream_t>(stream), nullptr);
}

int dhz_frames_u8_recover(const uint8_t* in, int64_t in_fs, int n, int H, int W, const dhz_params* p,
                          const double* airlight, uint8_t* out, int64_t out_fs, void* ws, size_t ws_bytes,
                          void* stream) {
  int rc = check_params(n, H, W, p);
  if (rc) return rc;
  if (n == 0) return DHZ_OK;
  const Layout L = make_layout(n, H, W, p);
  if ((rc = frames_check(in, in_fs, n, H, W, p, out, out_fs, airlight, ws, ws_bytes, L))) return rc;
  return frames_recover(in, in_fs, n, H, W, p, airlight, out, out_fs, static_cast<uint8_t*>(ws), L,
                        reinterpret_cast<cudaStream_t>(stream), nullptr);
}

/* ----------------------------------------------------------- resize path ---- */

namespace {

struct RLayout {
  int64_t hist, zero_end, sel, bal, dark, total, dark_fs;
};

RLayout make_rlayout(int n, int H, int W, const dhz_params* p) {
  RLayout L{};
  const int64_t npx = (int64_t)H * W;
  int64_t o = 0;
  auto take = [&](int64_t bytes) {
    const int64_t at = o;
    o = align_up(o + bytes);
    return at;
  };
  L.hist = take(4LL * dhz::kResizeBuckets * n);
  L.zero_end = o;
  L.sel = take(4LL * n * std::max<int64_t>(1, p->top_k));
  L.bal = p->balance ? take((int64_t)dhz::resize_balance_ws_bytes(n)) : -1;
  L.dark_fs = 8 * npx;
  L.dark = take(L.dark_fs * n);
  L.total = o;
  return L;
}

int check_resize(int n, int h, int w, int H, int W, const dhz_params* p) {
  int rc = check_params(n, H, W, p);
  if (rc) return rc;
  if (h < 1 || w < 1) return fail(DHZ_E_INVALID, "empty source frame %dx%d", w, h);
  if ((int64_t)h * w > 0x7FFFFFFFLL) return fail(DHZ_E_INVALID, "source frame too large");
  if (p->mode != 0) return fail(DHZ_E_UNSUPPORTED, "the resize path runs video mode only");
  if (p->patch_radius > dhz::kResizeMaxRadius)
    return fail(DHZ_E_UNSUPPORTED, "patch_radius %d above %d on the resize path", p->patch_radius,
                dhz::kResizeMaxRadius);
  return DHZ_OK;
}

dhz::ResizeGeo make_geo(int h, int w, int H, int W) {
  dhz::ResizeGeo g;
  g.h = h;
  g.w = w;
  g.H = H;
  g.W = W;
  g.sy = (double)h / (double)H;  // pipeline/imageops: h / height, w / width (IEEE division)
  g.sx = (double)w / (double)W;
  return g;
}

}  // namespace

size_t dhz_frames_resize_u8_workspace(int n, int h, int w, int height, int width, const dhz_params* p) {
  if (check_resize(std::max(n, 0), h, w, height, width, p) != DHZ_OK) return 0;
  return (size_t)make_rlayout(n, height, width, p).total;
}

int dhz_frames_resize_u8_layout(int n, int h, int w, int height, int width, const dhz_params* p, int64_t* off) {
  int rc = check_resize(n, h, w, height, width, p);
  if (rc) return rc;
  if (!off) return fail(DHZ_E_INVALID, "offsets is NULL");
  const RLayout L = make_rlayout(n, height, width, p);
  off[0] = L.dark;
  off[1] = L.dark_fs;
  off[2] = L.sel;
  off[3] = -1;
  off[4] = L.total;
  return DHZ_OK;
}

namespace {
int resize_check(const uint8_t* in, int64_t in_fs, int n, int h, int w, int H, int W, const void* out,
                 int64_t out_fs, const double* airlight, void* ws, size_t ws_bytes, const RLayout& L) {
  if (!in || !out || !airlight) return fail(DHZ_E_INVALID, "NULL array argument");
  if (in_fs < 3LL * h * w || out_fs < 3LL * H * W) return fail(DHZ_E_INVALID, "frame stride smaller than a frame");
  if (!ws || (int64_t)ws_bytes < L.total)
    return fail(DHZ_E_WORKSPACE, "workspace too small: need %lld bytes, got %zu", (long long)L.total, ws_bytes);
  return DHZ_OK;
}

int resize_airlight(const uint8_t* in, int64_t in_fs, int n, const dhz::ResizeGeo& g, const dhz_params* p,
                    double* airlight, uint8_t* base, const RLayout& L, cudaStream_t st, void* const* events) {
  auto mark = [&](int i) { record_stage_event(events, i, st); };
  double* dark = reinterpret_cast<double*>(base + L.dark);
  uint32_t* hist = reinterpret_cast<uint32_t*>(base + L.hist);
  uint32_t* sel = reinterpret_cast<uint32_t*>(base + L.sel);
  mark(0);
  cudaError_t e = cudaMemsetAsync(base, 0, (size_t)L.zero_end, st);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  e = dhz::resize_dark(in, in_fs, n, g, p->patch_radius, dark, hist, st);
  if (e != cudaSuccess) return cuda_fail(e, "resize_dark");
  mark(1);
  e = dhz::resize_select(in, in_fs, n, g, dark, hist, p->top_k, p->alpha, sel, airlight, st);
  if (e != cudaSuccess) return cuda_fail(e, "resize_select");
  mark(2);
  return DHZ_OK;
}

int resize_recover_stage(const uint8_t* in, int64_t in_fs, int n, const dhz::ResizeGeo& g, const dhz_params* p,
                         const double* airlight, uint8_t* out, int64_t out_fs, uint8_t* base, const RLayout& L,
                         cudaStream_t st, void* const* events) {
  record_stage_event(events, 3, st);
  cudaError_t e = dhz::resize_recover(in, in_fs, n, g, airlight, p->omega, p->t_min, p->thresholds, p->gamma,
                                      p->balance != 0, p->balance ? base + L.bal : nullptr, out, out_fs, st);
  if (e != cudaSuccess) return cuda_fail(e, "resize_recover");
  record_stage_event(events, 4, st);
  return DHZ_OK;
}
}  // namespace

int dhz_frames_resize_u8(const uint8_t* in, int64_t in_fs, int n, int h, int w, int H, int W, const dhz_params* p,
                         uint8_t* out, int64_t out_fs, double* airlight, void* ws, size_t ws_bytes, void* stream,
                         void* const* events) {
  int rc = check_resize(n, h, w, H, W, p);
  if (rc) return rc;
  if (n == 0) return DHZ_OK;
  const RLayout L = make_rlayout(n, H, W, p);
  if ((rc = resize_check(in, in_fs, n, h, w, H, W, out, out_fs, airlight, ws, ws_bytes, L))) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const dhz::ResizeGeo g = make_geo(h, w, H, W);
  uint8_t* base = static_cast<uint8_t*>(ws);
  if ((rc = resize_airlight(in, in_fs, n, g, p, airlight, base, L, st, events))) return rc;
  return resize_recover_stage(in, in_fs, n, g, p, airlight, out, out_fs, base, L, st, events);
}

int dhz_frames_resize_u8_airlight(const uint8_t* in, int64_t in_fs, int n, int h, int w, int H, int W,
                                  const dhz_params* p, double* airlight, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_resize(n, h, w, H, W, p);
  if (rc) return rc;
  if (n == 0) return DHZ_OK;
  const RLayout L = make_rlayout(n, H, W, p);
  if ((rc = resize_check(in, in_fs, n, h, w, H, W, airlight, 3LL * H * W, airlight, ws, ws_bytes, L))) return rc;
  return resize_airlight(in, in_fs, n, make_geo(h, w, H, W), p, airlight, static_cast<uint8_t*>(ws), L,
                         reinterpret_cast<cudaStream_t>(stream), nullptr);
}

int dhz_frames_resize_u8_recover(const uint8_t* in, int64_t in_fs, int n, int h, int w, int H, int W,
                                 const dhz_params* p, const double* airlight, uint8_t* out, int64_t out_fs, void* ws,
                                 size_t ws_bytes, void* stream) {
  int rc = check_resize(n, h, w, H, W, p);
  if (rc) return rc;
  if (n == 0) return DHZ_OK;
  const RLayout L = make_rlayout(n, H, W, p);
  if ((rc = resize_check(in, in_fs, n, h, w, H, W, out, out_fs, airlight, ws, ws_bytes, L))) return rc;
  return resize_recover_stage(in, in_fs, n, make_geo(h, w, H, W), p, airlight, out, out_fs,
                              static_cast<uint8_t*>(ws), L, reinterpret_cast<cudaStream_t>(stream), nullptr);
}

}  // extern "C"
