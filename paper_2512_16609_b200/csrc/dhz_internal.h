// Internal (C++) interfaces between the kernel translation units and the C ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include <utility>

namespace dhz {

// Kernel launch with programmatic dependent launch (PDL) on the same stream: the
// kernel may begin launching while the previous kernel drains (it must call
// pdl_wait() before touching predecessor data).  pdl = false: a plain launch.
bool pdl_enabled();  // DHZ_PDL=0 turns programmatic dependent launch off (A/B measurements)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Set the thread-local message returned by dhz_last_error(); return `code`.
int abi_fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int abi_cuda_fail(cudaError_t e, const char* where);

// Per-frame top-K selection state, one record per frame in the workspace.
struct FrameSel {
  uint32_t reserved;
  uint32_t mode;       // kSelFast / kSelFull / kSelAll
  uint32_t T;          // threshold (K-th largest dark value)
  uint32_t above;      // # pixels with dark > T
  uint32_t ticket;     // last-block counters
  uint32_t ticket2;
  uint32_t pad[2];
};
enum : uint32_t { kSelFast = 0, kSelFull = 1, kSelAll = 2 };

// K1: dark map (u8) + per-frame max.  dark_fs/in_fs are byte strides between frames.
cudaError_t dark_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, uint8_t* dark,
                    int64_t dark_fs, uint32_t* frame_max /* [n], zeroed by the caller */,
                    uint32_t* unit_max /* [n][ceil(H/16)][ceil(W/32)], zeroed by the caller */,
                    cudaStream_t st);
bool dark_rows_supported(int r, int W, int64_t in_fs, int64_t dark_fs, const void* in, const void* dark);
cudaError_t dark_rows(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, uint8_t* dark,
                      int64_t dark_fs, uint32_t* frame_max, uint32_t* unit_max, cudaStream_t st);
size_t dark_u8_max_smem(int r);

// K2/K3: ordered top-K select on the u8 dark map and the sequential fp64 airlight sum.
struct SelectWs {
  FrameSel* sel;         // [n]
  uint32_t* frame_max;   // [n]  (K1 output)
  uint32_t* unit_max;    // [n][ceil(H/16)][ceil(W/32)] max dark value per unit (K1 output)
  uint32_t* row_hist;    // [n][H][16] pixels per row at level max-j, zeroed by the caller
  uint32_t* frame_hist;  // [n][16], zeroed by the caller
  uint32_t* hist256;     // [n][256] full level histogram (fallback frames only), zeroed by the caller
  uint32_t* full_list;   // [n + 1]: count, then the frames on the fallback path; zeroed by the caller
  uint32_t* row_info;    // [n][H][4] = above, ties, above_prefix, tie_prefix
  uint32_t* sel_idx;     // [n][K] selected flat indices in summation order
  int H, W;
};
cudaError_t select_u8(const uint8_t* dark, int64_t dark_fs, const uint8_t* in, int64_t in_fs, int n, int64_t npx,
                      int64_t K, double alpha, const SelectWs& ws, double* airlight /* [n][3] */, cudaStream_t st);

// K5/K6: per-frame recovery LUT and the LUT apply pass.
cudaError_t build_lut_u8(int n, const double* airlight, double omega, double t_min, const double* thr,
                         double gamma /* only seeds the threshold search */, uint8_t* lut /* [n][3][kTri] */,
                         cudaStream_t st);
// Image mode: fused guided filter + recovery on u8 frames (guided_u8.cu).
constexpr int kGuidedMaxRadius = 255;  // 2r < 512 columns of the wide strip
size_t guided_ws_bytes(int n, int H, int W, int r, bool balance);
cudaError_t guided_recover_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, double eps,
                              const double* airlight, double omega, double t_min, const double* thr, double gamma,
                              bool balance, uint8_t* out, int64_t out_fs, void* ws, cudaStream_t st);

// Image mode, one-pass guided filter with exact integer box sums (guided_fused.cu),
// radius <= kFusedMaxRadius; the strip kernels above cover larger radii.
constexpr int kFusedMaxRadius = 63;
bool guided_fused_ok(int H, int W, int r);
bool guided_use_fused(int H, int W, int r);
int guided_path(int H, int W, int r);  // 0 strip kernels, 1 one-pass exact, 2 two-pass exact
size_t guided_fused_ws_bytes(int n, int H, int W, int r, bool balance);
cudaError_t guided_fused_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, double eps,
                            const double* airlight, double omega, double t_min, const double* thr, double gamma,
                            bool balance, uint8_t* out, int64_t out_fs, void* ws, cudaStream_t st);
// Two-pass form of the same exact filter (pass 1 writes the fixed-point a, b; pass 2
// boxes them): the same bytes as guided_fused_u8.
size_t guided_x_ws_bytes(int n, int H, int W, int r, bool balance);
cudaError_t guided_x_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, double eps,
                        const double* airlight, double omega, double t_min, const double* thr, double gamma,
                        bool balance, uint8_t* out, int64_t out_fs, void* ws, cudaStream_t st);
// Gray-world apply: bytes from t~ (fp64 [n][npx]), airlight and per-frame channel
// thresholds / gains (balance_thresholds below).
cudaError_t guided_apply(const uint8_t* in, int64_t in_fs, int n, int64_t npx, const double* t,
                         const double* airlight, const double* thr, const float* gains, double gamma, uint8_t* out,
                         int64_t out_fs, cudaStream_t st);

// Gray-world balance from per-CTA channel sums of the gamma values (part[n][nparts][3]):
// per frame and channel the gains and the 256 exact byte thresholds on the recovered
// value (thr[n][3][256], thr[.][.][0] = -1, +inf for unreachable levels); gains[n][3]
// (fp32) only seed the threshold walk.
cudaError_t balance_thresholds(const double* part, int nparts, int n, int64_t npx, double gamma, double* thr,
                               float* gains, cudaStream_t st);

// Default video mode: frames resized (fp64 bilinear, recomputed from the u8 input
// wherever needed) and dehazed at the working size (resize_u8.cu).
constexpr int kResizeMaxRadius = 32;
constexpr int kResizeBuckets = 4097;  // floor(dark * 4096) for dark in [0, 1]
constexpr int kResizeSumParts = 64;   // CTAs per frame of the balance sums pass
struct ResizeGeo {
  int h, w;        // source frame
  int H, W;        // working size (resize_to)
  double sy, sx;   // h / H, w / W (the reference's Python float divisions)
};
cudaError_t resize_dark(const uint8_t* in, int64_t in_fs, int n, const ResizeGeo& g, int r, double* dark,
                        uint32_t* hist /* [n][kResizeBuckets], zeroed by the caller */, cudaStream_t st);
cudaError_t resize_select(const uint8_t* in, int64_t in_fs, int n, const ResizeGeo& g, const double* dark,
                          const uint32_t* hist, int64_t K, double alpha, uint32_t* sel /* [n][K] */,
                          double* airlight, cudaStream_t st);
size_t resize_balance_ws_bytes(int n);
cudaError_t resize_recover(const uint8_t* in, int64_t in_fs, int n, const ResizeGeo& g, const double* airlight,
                           double omega, double t_min, const double* thr, double gamma, bool balance,
                           void* bal_ws, uint8_t* out, int64_t out_fs, cudaStream_t st);

// Gray-world balanced LUT (g table, per-frame channel sums, gains); ws: balance_ws_bytes(n).
size_t balance_ws_bytes(int n);
cudaError_t build_lut_balanced_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, const double* airlight,
                                  double omega, double t_min, double gamma, uint8_t* lut, void* ws,
                                  cudaStream_t st);
cudaError_t recover_lut_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, const uint8_t* lut,
                           uint8_t* out, int64_t out_fs, cudaStream_t st);

}  // namespace dhz
