// Internal (C++) interfaces between the kernel translation units and the C ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace dhz {

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
                    uint32_t* band_max /* [n][ceil(H/16)], zeroed by the caller */, cudaStream_t st);
bool dark_rows_supported(int r, int W, int64_t in_fs, int64_t dark_fs, const void* in, const void* dark);
cudaError_t dark_rows(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, uint8_t* dark,
                      int64_t dark_fs, uint32_t* frame_max, uint32_t* band_max, cudaStream_t st);
size_t dark_u8_max_smem(int r);

// K2..K4: ordered top-K select on the u8 dark map and the sequential fp64 airlight sum.
struct SelectWs {
  FrameSel* sel;        // [n]
  uint32_t* frame_max;  // [n]  (K1 output)
  uint32_t* band_max;   // [n][ceil(H/16)] max dark value per 16-row band (K1 output)
  int H, W;
  uint32_t* seg_hist;   // [n][S][16]
  uint32_t* seg_full;   // [n][S][256]   (fallback path)
  uint32_t* seg_meta;   // [n][S][4] = above_cnt, tie_cnt, above_off, tie_off
  uint32_t* sel_idx;    // [n][K]
  int S;                // segments per frame
};
cudaError_t select_u8(const uint8_t* dark, int64_t dark_fs, int n, int64_t npx, int64_t K,
                      const SelectWs& ws, cudaStream_t st);
cudaError_t airlight_sum_u8(const uint8_t* in, int64_t in_fs, int n, int64_t npx, int64_t K, double alpha,
                            const SelectWs& ws, double* airlight /* [n][3] */, cudaStream_t st);

// K5/K6: per-frame recovery LUT and the LUT apply pass.
cudaError_t build_lut_u8(int n, const double* airlight, double omega, double t_min, const double* thr,
                         uint8_t* lut /* [n][3][kTri] */, cudaStream_t st);
cudaError_t recover_lut_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, const uint8_t* lut,
                           uint8_t* out, int64_t out_fs, cudaStream_t st);

}  // namespace dhz
