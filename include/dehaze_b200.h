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

/* Byte offsets inside the workspace after dhz_frames_u8 returned (valid until the
 * workspace is reused): [0] dark map u8 (n x H*W, frame stride [1]),
 * [2] selected airlight pixel indices uint32 (n x K, in summation order),
 * [3] transmission map (image mode: float64, n x H*W; video mode: unused, -1),
 * [4] total workspace bytes. */
int dhz_frames_u8_layout(int n, int height, int width, const dhz_params* p, int64_t* offsets5);

#ifdef __cplusplus
}
#endif

#endif /* DEHAZE_B200_H */
