// K1 — dark channel of interleaved u8 RGB frames (channel min + (2r+1)^2 erosion).
//
// Replaces estimation.py:35-43 (channel_min, dark_channel) and morphology.py:17-73
// (_running_min_rows/_cols, min_filter) of the reference.  On the u8 grid every
// reference value is k/255 and min only selects, so the u8 dark map is bit-exact
// (dark_f64 == dark_u8 / 255.0 exactly).  Replicate borders are equivalent to
// clamping the window to the image, which is what the +inf (0xFF) fill does.
//
// Tile: 256 output columns x 64 output rows per CTA; halo of HP (>= r, multiple
// of 16) columns and r rows.  Loads are 48-byte (16-pixel) units of three
// 128-bit LDGs; the min filter is done vertically first (aligned words, sliding
// doubling in registers), then horizontally on bytes (SIMD doubling with funnel
// shifts).  Each CTA also folds its max into the per-frame max used by the
// top-K select (select_u8.cu).
#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

constexpr int kSW = 256;     // output columns per tile
constexpr int kBH = 64;      // output rows per tile
constexpr int kRun = 16;     // output rows per thread in the vertical pass
constexpr int kThreads = 256;

__host__ __device__ constexpr int halo_px(int r) { return ((r + 15) / 16) * 16; }

// Load phase: fill C[v][0..LW) with the channel-min bytes of image rows
// y0 - r + v (0xFF outside the image).
template <bool VEC>
__device__ __forceinline__ void load_cmin_tile(const uint8_t* __restrict__ frame, int H, int W, int r,
                                               int x0, int y0, int HP, int LW, int rows,
                                               uint8_t* __restrict__ C) {
  const int units_per_row = LW / 16;
  const int total = rows * units_per_row;
  for (int it = threadIdx.x; it < total; it += kThreads) {
    const int v = it / units_per_row;
    const int u = it - v * units_per_row;
    const int y = y0 - r + v;
    const int x = x0 - HP + 16 * u;
    uint32_t c[4];
    if (y < 0 || y >= H) {
      c[0] = c[1] = c[2] = c[3] = 0xFFFFFFFFu;
    } else {
      const uint8_t* row = frame + (int64_t)y * W * 3;
      if (VEC && x >= 0 && x + 16 <= W) {
        const uint4 a = ldg_v4(row + 3 * x);
        const uint4 b = ldg_v4(row + 3 * x + 16);
        const uint4 d = ldg_v4(row + 3 * x + 32);
        const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
        cmin16(w, c);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t word = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int px = x + 4 * q + k;
            uint32_t m = 0xFFu;
            if (px >= 0 && px < W) {
              const uint8_t* p = row + 3 * px;
              m = min(min((uint32_t)p[0], (uint32_t)p[1]), (uint32_t)p[2]);
            }
            word |= m << (8 * k);
          }
          c[q] = word;
        }
      }
    }
    *reinterpret_cast<uint4*>(C + v * LW + 16 * u) = make_uint4(c[0], c[1], c[2], c[3]);
  }
}

// Vertical sliding min over L = 2R+1 rows for one column word and kRun output rows,
// by power-of-two doubling in registers.  R is a compile-time radius.
template <int R>
__device__ __forceinline__ void vmin_run_static(const uint8_t* __restrict__ C, int LW, int cw, int j0,
                                                uint8_t* __restrict__ V) {
  constexpr int L = 2 * R + 1;
  constexpr int N = kRun + 2 * R;
  uint32_t m[N];
#pragma unroll
  for (int k = 0; k < N; ++k) m[k] = *reinterpret_cast<const uint32_t*>(C + (j0 + k) * LW + 4 * cw);
  // m[k] currently = min over window of length P starting at row k (P = 1).
  int P = 1;
#pragma unroll
  for (int lvl = 0; lvl < 6; ++lvl) {
    if (2 * P > L) break;
#pragma unroll
    for (int k = 0; k + P < N; ++k) m[k] = vmin4(m[k], m[k + P]);
    P *= 2;
  }
#pragma unroll
  for (int j = 0; j < kRun; ++j) {
    const uint32_t o = vmin4(m[j], m[j + L - P]);
    *reinterpret_cast<uint32_t*>(V + (j0 + j) * LW + 4 * cw) = o;
  }
}

__device__ __forceinline__ void vmin_run_dynamic(const uint8_t* __restrict__ C, int LW, int cw, int j0,
                                                 int r, uint8_t* __restrict__ V) {
  const int L = 2 * r + 1;
  for (int j = 0; j < kRun; ++j) {
    uint32_t o = 0xFFFFFFFFu;
    for (int k = 0; k < L; ++k) o = vmin4(o, *reinterpret_cast<const uint32_t*>(C + (j0 + j + k) * LW + 4 * cw));
    *reinterpret_cast<uint32_t*>(V + (j0 + j) * LW + 4 * cw) = o;
  }
}

__device__ __forceinline__ uint32_t word_at_byte(const uint32_t* m, int b) {
  const int i = b >> 2, s = b & 3;
  return s ? funnel_bytes(m[i], m[i + 1], s) : m[i];
}

// Horizontal sliding min over L = 2R+1 bytes for 32 output bytes (8 words) of one
// V row.  Output byte o of the chunk is centred at V byte HP + 32*chunk + o.
template <int R>
__device__ __forceinline__ void hmin_chunk_static(const uint8_t* __restrict__ Vrow, int HP, int chunk,
                                                  uint32_t (&out)[8]) {
  constexpr int L = 2 * R + 1;
  constexpr int HW = (R + 3) / 4;       // halo words each side
  constexpr int NW = 8 + 2 * HW + 1;    // +1 so funnel reads stay in range
  constexpr int S0 = 4 * HW - R;        // window start of output byte 0, relative to m[0]
  uint32_t m[NW];
  const uint32_t* src = reinterpret_cast<const uint32_t*>(Vrow + HP + 32 * chunk) - HW;
#pragma unroll
  for (int k = 0; k < NW; ++k) m[k] = src[k];
  int P = 1;
#pragma unroll
  for (int lvl = 0; lvl < 6; ++lvl) {
    if (2 * P > L) break;
    // m_2P[i] = min(m_P[i], m_P shifted by P bytes)
#pragma unroll
    for (int k = 0; k < NW - 1; ++k) {
      const int b = 4 * k + P;
      uint32_t sh;
      if ((P & 3) == 0) {
        sh = (k + (P >> 2) < NW) ? m[k + (P >> 2)] : 0xFFFFFFFFu;
      } else {
        const int i = b >> 2;
        sh = (i + 1 < NW) ? funnel_bytes(m[i], m[i + 1], b & 3) : 0xFFFFFFFFu;
      }
      m[k] = vmin4(m[k], sh);
    }
    P *= 2;
  }
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const uint32_t a = word_at_byte(m, S0 + 4 * w);
    const uint32_t b = word_at_byte(m, S0 + 4 * w + L - P);
    out[w] = vmin4(a, b);
  }
}

__device__ __forceinline__ void hmin_chunk_dynamic(const uint8_t* __restrict__ Vrow, int HP, int chunk, int r,
                                                   uint32_t (&out)[8]) {
  const uint8_t* base = Vrow + HP + 32 * chunk;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    uint32_t word = 0;
    for (int k = 0; k < 4; ++k) {
      const int o = 4 * w + k;
      uint32_t m = 0xFFu;
      for (int d = -r; d <= r; ++d) m = min(m, (uint32_t)base[o + d]);
      word |= m << (8 * k);
    }
    out[w] = word;
  }
}

template <bool VEC, int R>
__global__ void __launch_bounds__(kThreads)
k_dark_u8(const uint8_t* __restrict__ in, int64_t in_fs, int H, int W, int r,
          uint8_t* __restrict__ dark, int64_t dark_fs, uint32_t* __restrict__ frame_max,
          uint32_t* __restrict__ unit_max) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int f = blockIdx.z;
  const int x0 = blockIdx.x * kSW;
  const int y0 = blockIdx.y * kBH;
  const int rr = (R > 0) ? R : r;
  const int HP = halo_px(rr);
  const int LW = kSW + 2 * HP;
  const int rows = kBH + 2 * rr;
  uint8_t* C = smem;
  uint8_t* V = smem + rows * LW;
  const uint8_t* frame = in + f * in_fs;

  load_cmin_tile<VEC>(frame, H, W, rr, x0, y0, HP, LW, rows, C);
  __syncthreads();

  // Vertical pass over all LW/4 column words (halo columns included).
  const int ncw = LW / 4;
  const int items_v = ncw * (kBH / kRun);
  for (int it = threadIdx.x; it < items_v; it += kThreads) {
    const int run = it / ncw;
    const int cw = it - run * ncw;
    if (R > 0)
      vmin_run_static<(R > 0 ? R : 1)>(C, LW, cw, run * kRun, V);
    else
      vmin_run_dynamic(C, LW, cw, run * kRun, rr, V);
  }
  __syncthreads();

  // Horizontal pass: 32 output bytes per item.
  uint32_t tmax = 0;
  const int items_h = kBH * (kSW / 32);
  uint8_t* dframe = dark + f * dark_fs;
  for (int it = threadIdx.x; it < items_h; it += kThreads) {
    const int j = it / (kSW / 32);
    const int chunk = it - j * (kSW / 32);
    const int y = y0 + j;
    if (y >= H) continue;
    uint32_t o[8];
    if (R > 0)
      hmin_chunk_static<(R > 0 ? R : 1)>(V + j * LW, HP, chunk, o);
    else
      hmin_chunk_dynamic(V + j * LW, HP, chunk, rr, o);
    const int x = x0 + 32 * chunk;
    const uint32_t tmax_before = tmax;
    tmax = 0;
    uint8_t* dst = dframe + (int64_t)y * W + x;
    if (VEC && x + 32 <= W) {
#pragma unroll
      for (int w = 0; w < 8; ++w) tmax = vmax4(tmax, o[w]);
      reinterpret_cast<uint4*>(dst)[0] = make_uint4(o[0], o[1], o[2], o[3]);
      reinterpret_cast<uint4*>(dst)[1] = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
      for (int w = 0; w < 8; ++w) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int px = x + 4 * w + k;
          if (px < W) {
            const uint32_t b = (o[w] >> (8 * k)) & 0xFFu;
            dst[4 * w + k] = (uint8_t)b;
            tmax = max(tmax, b);
          }
        }
      }
    }
    {
      const uint32_t cm = max(max(tmax & 0xFFu, (tmax >> 8) & 0xFFu), max((tmax >> 16) & 0xFFu, tmax >> 24));
      if (x < W)
        atomicMax(unit_max + ((int64_t)f * ((H + kBandH - 1) / kBandH) + y / kBandH) * ((W + kUnitW - 1) / kUnitW) +
                      x / kUnitW,
                  cm);
      tmax = vmax4(tmax, tmax_before);
    }
  }
  // fold the 4 byte lanes, then reduce over the block
  tmax = max(max(tmax & 0xFFu, (tmax >> 8) & 0xFFu), max((tmax >> 16) & 0xFFu, tmax >> 24));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
  __shared__ uint32_t wmax[kThreads / 32];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = tmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t m = 0;
    for (int i = 0; i < kThreads / 32; ++i) m = max(m, wmax[i]);
    atomicMax(frame_max + f, m);
  }
}

template <bool VEC, int R>
cudaError_t launch_dark(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, uint8_t* dark,
                        int64_t dark_fs, uint32_t* frame_max, uint32_t* unit_max, cudaStream_t st) {
  const int rr = R > 0 ? R : r;
  const int HP = halo_px(rr);
  const int LW = kSW + 2 * HP;
  const size_t smem = (size_t)(kBH + 2 * rr) * LW + (size_t)kBH * LW + 16;  // +16: funnel over-read pad
  auto kern = k_dark_u8<VEC, R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((W + kSW - 1) / kSW, (H + kBH - 1) / kBH, n);
  kern<<<grid, kThreads, smem, st>>>(in, in_fs, H, W, r, dark, dark_fs, frame_max, unit_max);
  return cudaGetLastError();
}

}  // namespace

size_t dark_u8_max_smem(int r) {
  const int HP = halo_px(r);
  const int LW = kSW + 2 * HP;
  return (size_t)(kBH + 2 * r) * LW + (size_t)kBH * LW + 16;
}

cudaError_t dark_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, uint8_t* dark,
                    int64_t dark_fs, uint32_t* frame_max, uint32_t* unit_max, cudaStream_t st) {
  if (dark_rows_supported(r, W, in_fs, dark_fs, in, dark))
    return dark_rows(in, in_fs, n, H, W, r, dark, dark_fs, frame_max, unit_max, st);
  const bool vec = (W % 16 == 0) && (in_fs % 16 == 0) && (dark_fs % 16 == 0) &&
                   ((uintptr_t)in % 16 == 0) && ((uintptr_t)dark % 16 == 0);
  if (vec) return launch_dark<true, 0>(in, in_fs, n, H, W, r, dark, dark_fs, frame_max, unit_max, st);
  if (r == 7) return launch_dark<false, 7>(in, in_fs, n, H, W, r, dark, dark_fs, frame_max, unit_max, st);
  return launch_dark<false, 0>(in, in_fs, n, H, W, r, dark, dark_fs, frame_max, unit_max, st);
}

}  // namespace dhz
