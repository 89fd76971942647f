/*
 * dehaze_b200.h — C ABI of the B200-native Hazedefy dehaze path (libdehaze_b200.so).
 *
 * The reference (/root/reference/pkg/src/dehaze) is a pure-Python package with no
 * FFI; its drop-in boundary is the public Python API exported by __init__.py:32-60.
 * This header is what that API's host mirror (paper_2512_16609_b200/, ctypes) binds.
 * Each entry point names the reference function(s) whose semantics it implements.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA storage);
 *    `stream` is a cudaStream_t (NULL = legacy default stream).  Calls enqueue work
 *    and return without synchronising.
 *  - Frames are interleaved RGB uint8, row-major (H, W, 3); `*_fs` arguments are the
 *    byte stride between consecutive frames of a batch.  float64 images are (H, W, 3)
 *    row-major, maps are (H, W) row-major.
 *  - The library never allocates device memory: callers pass a workspace sized by
 *    the matching *_workspace() query.
 *  - A batch call takes at most 65535 frames (DHZ_E_INVALID otherwise; split larger
 *    batches).  A frame's output never depends on the batch it arrives in.
 *  - Return value 0 = success; negative = error, message in dhz_last_error()
 *    (thread-local).  Argument validation with the reference's ValueError messages
 *    stays on the host side (paper_2512_16609_b200/validation.py); the C side only
 *    rejects what would be unsafe to launch.
 */
#ifndef DEHAZE_B200_H
#define DEHAZE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DHZ_OK 0
#define DHZ_E_INVALID (-1)
#define DHZ_E_CUDA (-2)
#define DHZ_E_WORKSPACE (-3)
#define DHZ_E_UNSUPPORTED (-4)

#define DHZ_ABI_VERSION 1

/* Pipeline parameters; mirrors DehazeParams (reference pipeline.py:52-114).  The host
 * resolves: top_k = max(1, floor(top_fraction * H * W)) (estimation.py:72),
 * balance = DehazeParams.balance_enabled() (pipeline.py:111-114), and the 256-entry
 * quantisation threshold table for `gamma` (paper_2512_16609_b200/quant.py). */
typedef struct dhz_params {
  int32_t mode;          /* 0 = video, 1 = image (guided-filter refinement)       */
  int32_t patch_radius;  /* dark-channel erosion radius r (window 2r+1)           */
  int64_t top_k;         /* K, number of airlight pixels                          */
  double alpha;          /* airlight damping                                      */
  double omega;          /* haze retention                                        */
  double t_min;          /* transmission floor                                    */
  int32_t guided_radius; /* guided-filter box radius (image mode)                 */
  int32_t balance;       /* 1 = gray-world balance                                */
  double guided_eps;     /* guided-filter regulariser                             */
  double gamma;          /* output gamma (informational; thresholds encode it)    */
  const double* thresholds; /* DEVICE, 256 doubles: thr[k] = smallest x in [0,1] whose
                               output byte is >= k (thr[0] unused)                 */
} dhz_params;

const char* dhz_last_error(void);
int dhz_abi_version(void);
/* Number of visible CUDA devices (>= 1) or DHZ_E_CUDA when there is none. */
int dhz_device_count(void);

/* ---------------------------------------------------------------------------
 * Fused u8 frame pipeline at native resolution.
 * Replaces dehaze_frame (pipeline.py:163-216) for u8 frames with resize a no-op,
 * video mode, i.e. the stages channel_min, min_filter, airlight, transmission,
 * recover, postprocess (gamma [+ gray-world]) and output, over a batch of frames
 * (process_stream, pipeline.py:232-308, minus host orchestration).
 *   in/out:   n frames, H x W x 3 u8; airlight: n x 3 doubles (device).
 * Image mode (p->mode == 1) adds the guided-filter refinement
 * (estimation.py:144-172, pipeline.py:197-203).
 * ------------------------------------------------------------------------- */
size_t dhz_frames_u8_workspace(int n, int height, int width, const dhz_params* p);
int dhz_frames_u8(const uint8_t* in, int64_t in_fs, int n, int height, int width, const dhz_params* p,
                  uint8_t* out, int64_t out_fs, double* airlight, void* ws, size_t ws_bytes, void* stream,
                  void* const* events);
/* events: NULL, or DHZ_N_EVENTS cudaEvent_t recorded on `stream` at: [0] start,
 * [1] after the dark channel (channel_min + min_filter), [2] after airlight,
 * [3] after transmission (image mode: + guided filter), [4] after recover +
 * postprocess + output.  Used for FrameTelemetry stage times. */
#define DHZ_N_EVENTS 5

/* The same pipeline in two halves, for the opt-in temporal stabilisation (the
 * airlight trace is smoothed between them; paper_2512_16609_b200 pipeline
 * `stabilise=`, not reference behaviour) and for multi-GPU runs that exchange the
 * trace first.  _airlight runs K1-K4 (channel_min, min_filter, estimate_airlight:
 * reference pipeline.py:182-190, estimation.py:46-84) and writes airlight (n x 3);
 * _recover runs the remaining stages (pipeline.py:192-216) from a CALLER-GIVEN
 * airlight.  dhz_frames_u8 == _airlight followed by _recover on the same workspace. */
int dhz_frames_u8_airlight(const uint8_t* in, int64_t in_fs, int n, int height, int width, const dhz_params* p,
                           double* airlight, void* ws, size_t ws_bytes, void* stream);
int dhz_frames_u8_recover(const uint8_t* in, int64_t in_fs, int n, int height, int width, const dhz_params* p,
                          const double* airlight, uint8_t* out, int64_t out_fs, void* ws, size_t ws_bytes,
                          void* stream);

/* Byte offsets inside the workspace after dhz_frames_u8 returned (valid until the
 * workspace is reused): [0] dark map u8 (n x H*W, frame stride [1]),
 * [2] selected airlight pixel indices uint32 (n x K, in summation order),
 * [3] image mode: guided-filter scratch (fp64 a, b maps of the last frame chunk);
 *     video mode: -1,
 * [4] total workspace bytes. */
int dhz_frames_u8_layout(int n, int height, int width, const dhz_params* p, int64_t* offsets5);

/* ---------------------------------------------------------------------------
 * Default video mode: the same stages with the frames first resized from
 * h x w to height x width (resize_to) by the reference's pixel-centre bilinear
 * filter in float64 (imageops.py:47-78, pipeline.py:175-180).  Replaces
 * dehaze_frame / process_stream with DehazeParams() (resize_to=(640, 480)) on
 * non-640x480 input.  p->mode must be 0 and p->top_k refers to height*width;
 * patch_radius <= 32.  out: n frames height x width x 3 u8.  Events as above
 * ([3] == [2]: no separate transmission stage).
 * ------------------------------------------------------------------------- */
size_t dhz_frames_resize_u8_workspace(int n, int h, int w, int height, int width, const dhz_params* p);
int dhz_frames_resize_u8(const uint8_t* in, int64_t in_fs, int n, int h, int w, int height, int width,
                         const dhz_params* p, uint8_t* out, int64_t out_fs, double* airlight, void* ws,
                         size_t ws_bytes, void* stream, void* const* events);
/* Two halves of dhz_frames_resize_u8, as for the native size above. */
int dhz_frames_resize_u8_airlight(const uint8_t* in, int64_t in_fs, int n, int h, int w, int height, int width,
                                  const dhz_params* p, double* airlight, void* ws, size_t ws_bytes, void* stream);
int dhz_frames_resize_u8_recover(const uint8_t* in, int64_t in_fs, int n, int h, int w, int height, int width,
                                 const dhz_params* p, const double* airlight, uint8_t* out, int64_t out_fs,
                                 void* ws, size_t ws_bytes, void* stream);
/* Offsets after dhz_frames_resize_u8: [0] dark map float64 (n x height*width,
 * frame stride [1] bytes), [2] selected indices uint32 (n x K, summation order),
 * [3] -1, [4] total workspace bytes. */
int dhz_frames_resize_u8_layout(int n, int h, int w, int height, int width, const dhz_params* p,
                                int64_t* offsets5);

/* ---------------------------------------------------------------------------
 * Multi-GPU (one process) and the opt-in airlight stabilisation.
 * Video batches shard by frame into contiguous blocks, one per device (frames are
 * independent: reference pipeline.py:257-260); the only exchange is the per-frame
 * airlight trace (reference StreamStats.airlight_trace, pipeline.py:279,308).
 * ------------------------------------------------------------------------- */
/* Device group for dhz_allgather_airlight: enables peer access (NVLink) between the
 * distinct devices; *comm receives an opaque handle.  A device may repeat (several
 * shards on one GPU). */
int dhz_comm_init(int ndev, const int* devices, void** comm);
int dhz_comm_destroy(void* comm);
/* All-gather of the per-device airlight blocks: device d holds counts[d] frames at
 * send[d] (counts[d] x 3 doubles, on device d); afterwards recv[d] (sum(counts) x 3
 * doubles on device d) holds every block in device order.  Enqueued on streams[d]
 * (cudaStream_t on device d), ordered after the work already on every source
 * stream; no host synchronisation. */
int dhz_allgather_airlight(void* comm, const double* const* send, const int* counts, double* const* recv,
                           void* const* streams);
/* Opt-in temporal stabilisation (north_star; NOT reference behaviour):
 * out[f] = lam * out[f-1] + (1 - lam) * trace[f] per channel, each product and sum
 * rounded once, out[-1] = carry (3 doubles) or out[0] = trace[0] when carry is NULL.
 * trace, out: n x 3 doubles (device, may alias only if equal); lam in [0, 1). */
int dhz_ema_airlight(const double* trace, int n, double lam, const double* carry, double* out, void* stream);

/* ---------------------------------------------------------------------------
 * float64 stage operations (reference public functions on float64 arrays; one
 * numpy operation = one IEEE rounding, so results match numpy bit for bit except
 * power() and the summation order of means / box sums).  Images are (H, W, 3),
 * maps (H, W); `n` counts elements, `npx` pixels.  Scratch buffers (`tmp`, `ws`)
 * are caller-allocated device memory of the stated size.
 * ------------------------------------------------------------------------- */
/* validation.py:32-72 helper: out3 = {all finite ? 1 : 0, min, max}; ws >= 3*1024 doubles */
int dhz_f64_stats(const double* x, int64_t n, double* out3, double* ws, void* stream);
/* imageops.py:18-21 u8_to_float */
int dhz_u8_to_f64(const uint8_t* in, int64_t n, double* out, void* stream);
/* imageops.py:24-36 float_to_u8 (clip, *255, +0.5, floor) */
int dhz_f64_to_u8(const double* in, int64_t n, uint8_t* out, void* stream);
/* imageops.py:39-44 to_grayscale */
int dhz_to_grayscale_f64(const double* img, int64_t npx, double* out, void* stream);
/* imageops.py:47-78 resize_bilinear; the _u8 variant fuses u8_to_float */
int dhz_resize_bilinear_f64(const double* in, int h, int w, int height, int width, double* out, void* stream);
int dhz_resize_bilinear_u8(const uint8_t* in, int h, int w, int height, int width, double* out, void* stream);
/* estimation.py:35-38 channel_min */
int dhz_channel_min_f64(const double* img, int64_t npx, double* out, void* stream);
/* morphology.py:63-73 min_filter (radius >= 1; tmp: H*W doubles) */
int dhz_min_filter_f64(const double* m, int height, int width, int radius, double* out, double* tmp, void* stream);
/* morphology.py:76-92 min_filter_naive / estimation.py:128-141 box_filter_naive: the
 * reference's per-pixel correctness references, as direct window scans (independent
 * of the separable kernels; radius >= 1) */
int dhz_min_filter_naive_f64(const double* m, int height, int width, int radius, double* out, void* stream);
int dhz_box_filter_naive_f64(const double* m, int height, int width, int radius, double* out, void* stream);
/* estimation.py:110-125 box_filter (radius >= 1; tmp: H*W doubles) */
int dhz_box_filter_f64(const double* m, int height, int width, int radius, double* out, double* tmp, void* stream);
/* estimation.py:144-172 guided_filter; floor_t > 0 also applies pipeline.py:203
 * max(q, t_min); ws: 7*H*W doubles */
int dhz_guided_filter_f64(const double* p, const double* guide, int height, int width, int radius, double eps,
                          double floor_t, double* out, double* ws, void* stream);
/* estimation.py:87-101 transmission_from_channel_min; airlight: 3 doubles (device) */
int dhz_transmission_f64(const double* cmin, int64_t npx, const double* airlight, double omega, double t_min,
                         double* out, void* stream);
/* recover.py:28-43 recover_radiance */
int dhz_recover_f64(const double* img, const double* airlight, const double* t, int64_t npx, double* out,
                    void* stream);
/* recover_radiance -> gamma_correct -> float_to_u8 fused, exact through the threshold table */
int dhz_recover_quant_f64(const double* img, const double* airlight, const double* t, int64_t npx,
                          const double* thresholds, uint8_t* out, void* stream);
/* recover.py:46-54 gamma_correct (gamma != 1; the caller copies for gamma == 1) */
int dhz_gamma_f64(const double* in, int64_t n, double gamma, double* out, void* stream);
/* recover.py:57-69 gray_world_balance; ws >= 3*256 + 4 doubles */
int dhz_gray_world_f64(const double* img, int64_t npx, double* out, double* ws, void* stream);
/* estimation.py:46-84 estimate_airlight on a float64 dark map: airlight (3 doubles) and the
 * K selected flat indices in summation order */
int dhz_airlight_f64(const double* img, const double* dark, int64_t npx, int64_t top_k, double alpha,
                     double* airlight, uint32_t* selected, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DEHAZE_B200_H */
