// K1 — dark channel of u8 RGB frames, row-major two-pass kernel (the fast path).
//
// Contract (reference estimation.py:35-43, morphology.py:17-73): dark =
// (2r+1)^2 erosion of the per-pixel channel minimum, window clamped to the
// image (== replicate padding for a min).  Bit-exact on the u8 grid.
//
// Tile: 480 output columns x 64 output rows, 256 threads (8 warps), ~37 KB
// of shared memory -> 5 CTAs / SM.
//  pass 1 (warp per row, rows y0-r .. y0+64+r): each lane streams 16 pixels
//    (3 coalesced 128-bit loads), forms their channel minima on 16-bit lanes,
//    borrows r pixels from each neighbour lane with shuffles and runs the
//    horizontal window min in registers (power-of-3 window growth on
//    VIMNMX3.U16x2, funnel shifts for odd offsets).  Lanes 0 and 31 only
//    supply halo, so a warp yields 480 pixels; the row goes to shared memory.
//  pass 2 (thread per 4 columns x 16 rows): vertical window min of the
//    shared rows in registers and a coalesced 4-byte store per row, plus the
//    max over each 16-row x 32-column unit (unit_max[], from per-item maxima)
//    and per frame (frame_max[]) that let the top-K select skip units that cannot
//    hold selected pixels.
#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched through the runtime)

#include <cstdlib>

#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

// ---- TMA row staging (DHZ_K1_TMA=1) ----
// Each warp owns one 1,536-byte stage and one mbarrier: lane 0 issues a
// cp.async.bulk.tensor (3-D map over [frame][row][3W/8 x u64]) for the warp's next row
// right after the current row has been copied from the stage into registers, so the
// stage plus the registers form the double buffer the LDG variant keeps in registers
// alone.  Out-of-frame bytes arrive as zeros and are replaced by the all-ones neutral.
constexpr int kTmaRowBytes = 1536;  // 32 lanes x 48 B (512 pixels)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_row(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(b))
      : "memory");
}

constexpr int kTW = kBandW;  // output columns per tile (30 lanes x 16 px)
constexpr int kBH = 64;    // output rows per tile (large batches)
constexpr int kBHSmall = 16;  // small batches (a frame or two): 4x the CTAs, each a quarter of the
                              // serial work — the halo rows it re-reads come from L2 and the
                              // launch is latency-bound anyway (one VGA frame: 16 -> 60 CTAs)
constexpr int kRun = kBandH;  // rows per pass-2 item (== unit height of unit_max)
constexpr int kThreads = 256;
#ifndef DHZ_K1_MINB
#define DHZ_K1_MINB 4  // resident CTAs per SM the register budget is sized for
#endif

template <int R, int BH = kBH>
struct RowGeo {
  static constexpr int L = 2 * R + 1;
  static constexpr int ROWS = BH + 2 * R;
  static constexpr int P = L >= 27 ? 27 : (L >= 9 ? 9 : (L >= 3 ? 3 : 1));
  static constexpr int HPR = (R + 1) / 2;        // neighbour pairs borrowed each side
  static constexpr int NP = 2 * HPR + 8 + 1;     // local pairs (+1 neutral pad)
  static constexpr size_t SMEM = (size_t)ROWS * kTW;
  static constexpr size_t STAGE_OFF = (SMEM + 127) / 128 * 128;  // TMA stages behind the row minima
  static constexpr size_t SMEM_TMA = STAGE_OFF + (size_t)(256 / 32) * kTmaRowBytes;
};

// Pipe balance.  Both passes are bound by the integer ALU pipe (~90 % busy in ncu,
// the FMA pipe ~10 %).  A pixel's value sits in the HIGH byte of its 16-bit lane with
// anything in the low byte: a 16-bit min or max then carries the min/max of the
// high bytes, so the channel split needs no masking (3 PRMT per pair, no LOP3) and
// pass 2 unpacks a shared-memory word w as the lane pairs (w << 8, w) — an IMAD.SHL
// on the FMA pipe and nothing — instead of two PRMTs (K1 0.578 -> 0.538 ms on C3).
// (Moving the 16-bit lane shifts to the FMA pipe as mad.hi(a, 2^16, b * 2^16)
// measured slower for every subset of them: 0.551-0.628 ms.)
template <int NP>
__device__ __forceinline__ uint32_t at(const uint32_t (&m)[NP], int px) {
  return (px & 1) ? shift1(m[px >> 1], m[(px >> 1) + 1]) : m[px >> 1];
}

// channel minimum of 16 pixels (48 bytes in 12 words) as 8 16x2 pairs, each pixel's
// value in the high byte of its lane (low byte: another channel's byte)
__device__ __forceinline__ void cmin16_pairs(const uint32_t (&w)[12], uint32_t (&c)[8]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t a = w[3 * q], b = w[3 * q + 1], d = w[3 * q + 2];
    // pixels 4q, 4q+1: R (a0, a3), G (a1, b0), B (a2, b1)
    c[2 * q] = min3(__byte_perm(a, a, 0x3300), __byte_perm(a, b, 0x4411), __byte_perm(a, b, 0x5522));
    // pixels 4q+2, 4q+3: R (b2, d1), G (b3, d2), B (d0, d3)
    c[2 * q + 1] = min3(__byte_perm(b, d, 0x5522), __byte_perm(b, d, 0x6633), __byte_perm(d, d, 0x3300));
  }
}
// high bytes of two lane pairs -> 4 bytes [lo.1, lo.3, hi.1, hi.3]
__device__ __forceinline__ uint32_t pack_hi(uint32_t lo, uint32_t hi) { return __byte_perm(lo, hi, 0x7531); }

template <int L, int N>
__device__ __forceinline__ void vert_levels(uint32_t (&v)[N]) {
  constexpr int P = L >= 27 ? 27 : (L >= 9 ? 9 : (L >= 3 ? 3 : 1));
  if (P >= 3) {
#pragma unroll
    for (int k = 0; k + 2 < N; ++k) v[k] = min3(v[k], v[k + 1], v[k + 2]);
  }
  if (P >= 9) {
#pragma unroll
    for (int k = 0; k + 6 < N; ++k) v[k] = min3(v[k], v[k + 3], v[k + 6]);
  }
  if (P >= 27) {
#pragma unroll
    for (int k = 0; k + 18 < N; ++k) v[k] = min3(v[k], v[k + 9], v[k + 18]);
  }
}
template <int L, int N>
__device__ __forceinline__ uint32_t vert_final(const uint32_t (&v)[N], int j) {
  constexpr int P = L >= 27 ? 27 : (L >= 9 ? 9 : (L >= 3 ? 3 : 1));
  if (L == P) return v[j];
  if (L <= 2 * P) return min2(v[j], v[j + L - P]);
  return min3(v[j], v[j + P], v[j + L - P]);
}

template <int R, bool TMA, int BH>
__global__ void __launch_bounds__(kThreads, R <= 8 ? DHZ_K1_MINB : 1)
k_dark_rows(const uint8_t* __restrict__ in, int64_t in_fs, int H, int W, uint8_t* __restrict__ dark,
            int64_t dark_fs, uint32_t* __restrict__ frame_max, uint32_t* __restrict__ unit_max,
            const __grid_constant__ CUtensorMap tmap) {
  using G = RowGeo<R, BH>;
  constexpr int L = G::L, P = G::P, HPR = G::HPR, NP = G::NP;
  extern __shared__ __align__(128) uint8_t hrow[];  // [ROWS][kTW] horizontal minima (+ TMA stages)
  const int f = blockIdx.z;
  const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * BH;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint8_t* frame = in + (int64_t)f * in_fs;

  // ---------------- pass 1: channel min + horizontal min, warp per row ----------------
  const int x = x0 - 16 + 16 * lane;  // first pixel of this lane
  const bool col_ok = x >= 0 && x < W;  // W % 16 == 0: a 16-px unit is fully in or out
  // register double buffering: row v+8's three 128-bit loads are in flight while
  // row v is reduced (the loop is otherwise bound by the load latency)
  // rows advance by 8 per iteration: walk a pointer instead of recomputing y*W*3
  const int64_t pitch8 = 3LL * W * (kThreads / 32);
  const uint8_t* src_row = frame + ((int64_t)(y0 - R + warp) * W + x) * 3;
  auto load_row = [&](int v, uint4& a, uint4& b, uint4& d) {
    const int y = y0 - R + v;
    if (v < G::ROWS && y >= 0 && y < H && col_ok) {
      a = ldg_v4(src_row);
      b = ldg_v4(src_row + 16);
      d = ldg_v4(src_row + 32);
    } else {
      a = b = d = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    }
    src_row += pitch8;
  };
  // TMA variant: the warp's stage and barrier; issue_row(v) arms the barrier and starts
  // the bulk copy of row v (rows outside the frame are not fetched)
  __shared__ __align__(8) uint64_t s_mbar[kThreads / 32];
  uint8_t* stage = hrow + G::STAGE_OFF + (size_t)warp * kTmaRowBytes;
  uint64_t* mbar = &s_mbar[warp];
  uint32_t parity = 0;
  auto row_ok = [&](int v) {
    const int y = y0 - R + v;
    return v < G::ROWS && y >= 0 && y < H;
  };
  auto issue_row = [&](int v) {
    if (lane == 0 && row_ok(v)) {
      mbar_expect_tx(mbar, kTmaRowBytes);
      tma_load_row(stage, &tmap, (x0 - 16) * 3 / 8, y0 - R + v, f, mbar);
    }
  };
  if (TMA) {
    if (lane == 0) {
      mbar_init(mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    issue_row(warp);
  }
  uint4 na, nb, nd;
  if (!TMA) load_row(warp, na, nb, nd);
  for (int v = warp; v < G::ROWS; v += kThreads / 32) {
    uint4 a, b, d;
    if (TMA) {
      a = b = d = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      if (row_ok(v)) {  // warp-uniform
        mbar_wait(mbar, parity);
        parity ^= 1;
        if (col_ok) {
          const uint4* sp = reinterpret_cast<const uint4*>(stage + 48 * lane);
          a = sp[0];
          b = sp[1];
          d = sp[2];
        }
      }
      __syncwarp();  // every lane has read the stage before it is refilled
      issue_row(v + kThreads / 32);
    } else {
      a = na, b = nb, d = nd;
      load_row(v + kThreads / 32, na, nb, nd);
    }
    uint32_t c[8];
    {
      const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
      cmin16_pairs(w, c);  // all-ones words (outside the frame) stay all-ones
    }
    // local pairs: [HPR from the left lane][8 own][HPR from the right lane][pad]
    uint32_t m[NP];
#pragma unroll
    for (int k = 0; k < HPR; ++k) {
      m[k] = __shfl_up_sync(0xffffffffu, c[8 - HPR + k], 1);
      m[HPR + 8 + k] = __shfl_down_sync(0xffffffffu, c[k], 1);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) m[HPR + k] = c[k];
    m[NP - 1] = 0xFFFFFFFFu;
    if (P >= 3) {
#pragma unroll
      for (int p = 0; p + 1 < NP; ++p) m[p] = min3(m[p], shift1(m[p], m[p + 1]), m[p + 1]);
    }
    if (P >= 9) {
#pragma unroll
      for (int p = 0; p + 3 < NP; ++p) m[p] = min3(m[p], shift1(m[p + 1], m[p + 2]), m[p + 3]);
    }
    if (P >= 27) {
#pragma unroll
      for (int p = 0; p + 9 < NP; ++p) m[p] = min3(m[p], shift1(m[p + 4], m[p + 5]), m[p + 9]);
    }
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t pr[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int s = 2 * HPR + 4 * q + 2 * h - R;  // local window start of the pair's lane 0
        if (L == P) pr[h] = at(m, s);
        else if (L <= 2 * P) pr[h] = min2(at(m, s), at(m, s + L - P));
        else pr[h] = min3(at(m, s), at(m, s + P), at(m, s + L - P));
      }
      o[q] = pack_hi(pr[0], pr[1]);
    }
    if (lane >= 1 && lane <= 30)
      *reinterpret_cast<uint4*>(hrow + (size_t)v * kTW + 16 * (lane - 1)) = make_uint4(o[0], o[1], o[2], o[3]);
  }
  __syncthreads();

  // ---------------- pass 2: vertical min, thread per 4 columns x 16 rows ----------------
  constexpr int NG = kTW / 4;                 // 120 column groups
  static_assert(BH % kRun == 0, "tiles hold whole runs");
  static_assert(NG % 8 == 0 && kTW % kUnitW == 0 && kRun == kBandH, "unit maxima: 8 groups of 4 columns");
  static_assert(((kTW / kUnitW) * (BH / kRun) + 31) / 32 * 32 <= kThreads, "one thread per unit");
  constexpr int N = kRun + 2 * R;
  __shared__ __align__(16) uint32_t item_max[NG * (BH / kRun)];
  for (int it = threadIdx.x; it < NG * (BH / kRun); it += kThreads) {
    const int run = it / NG, g = it - run * NG;
    const int j0 = run * kRun;
    const int xo = x0 + 4 * g;
    uint32_t lo[N], hi[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(hrow + (size_t)(j0 + k) * kTW + 4 * g);
      lo[k] = w << 8;  // pixels 0, 2 in the high bytes
      hi[k] = w;       // pixels 1, 3
    }
    vert_levels<L, N>(lo);
    vert_levels<L, N>(hi);
    uint32_t mx = 0;
    if (xo < W) {
      uint32_t* dst = reinterpret_cast<uint32_t*>(dark + (int64_t)f * dark_fs + (int64_t)(y0 + j0) * W + xo);
      const int wstep = W >> 2;  // row pitch in words (W % 16 == 0 on this path)
      if (y0 + j0 + kRun <= H) {  // whole run inside the frame: no per-row checks
#pragma unroll
        for (int j = 0; j < kRun; ++j) {
          const uint32_t a = vert_final<L, N>(lo, j), b = vert_final<L, N>(hi, j);
          dst[j * wstep] = __byte_perm(a, b, 0x7351);
          mx = max3u(mx, a, b);
        }
      } else {
#pragma unroll
        for (int j = 0; j < kRun; ++j) {
          const uint32_t a = vert_final<L, N>(lo, j), b = vert_final<L, N>(hi, j);
          if (y0 + j0 + j < H) {
            dst[j * wstep] = __byte_perm(a, b, 0x7351);
            mx = max3u(mx, a, b);
          }
        }
      }
    }
    item_max[it] = max((mx >> 8) & 0xFFu, mx >> 24);
  }
  __syncthreads();
  // unit maxima (8 column groups of 4 = 32 columns) and the frame maximum
  constexpr int NU = kTW / kUnitW;  // 15 units per tile row
  constexpr int NUT = NU * (BH / kRun);
  if (threadIdx.x < (NUT + 31) / 32 * 32) {  // whole warps: the shuffles below need them
    uint32_t um = 0;
    if (threadIdx.x < NUT) {
      const int run = threadIdx.x / NU, u = threadIdx.x - run * NU;
      const uint4 a = *reinterpret_cast<const uint4*>(&item_max[run * NG + 8 * u]);
      const uint4 b = *reinterpret_cast<const uint4*>(&item_max[run * NG + 8 * u + 4]);
      um = max(max(max(a.x, a.y), max(a.z, a.w)), max(max(b.x, b.y), max(b.z, b.w)));
      const int xu = x0 + kUnitW * u, yr = y0 + run * kRun;
      if (xu < W && yr < H)
        unit_max[((int64_t)f * ((H + kBandH - 1) / kBandH) + yr / kBandH) * ((W + kUnitW - 1) / kUnitW) +
                 xu / kUnitW] = um;
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) um = max(um, __shfl_xor_sync(0xffffffffu, um, sh));
    if (lane == 0 && um) atomicMax(frame_max + f, um);
  }
  pdl_trigger();  // the select chain (PDL) may start launching
}

// Tensor map over the batch as [n][H][3W/8] u64 (row pitch 3W, frame pitch in_fs; both
// multiples of 16 on this path), box = one 1,536-byte row segment.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
bool make_row_map(const uint8_t* in, int64_t in_fs, int n, int H, int W, CUtensorMap* map) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(3LL * W / 8), (cuuint64_t)H, (cuuint64_t)n};
  const cuuint64_t strides[2] = {(cuuint64_t)(3LL * W), (cuuint64_t)in_fs};
  const cuuint32_t box[3] = {kTmaRowBytes / 8, 1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint8_t*>(in), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool use_tma() {  // read per launch (tests switch it inside one process)
  const char* e = std::getenv("DHZ_K1_TMA");
  return e && e[0] == '1';
}

bool small_tiles(int n, int H, int W) {  // fewer 64-row tiles than two per SM: cut them in four
  if (const char* e = std::getenv("DHZ_K1_BH")) return std::atoi(e) == kBHSmall;  // tests force either
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int64_t)n * ((W + kTW - 1) / kTW) * ((H + kBH - 1) / kBH) < 2LL * sms;
}

template <int R>
cudaError_t launch(const uint8_t* in, int64_t in_fs, int n, int H, int W, uint8_t* dark, int64_t dark_fs,
                   uint32_t* frame_max, uint32_t* unit_max, cudaStream_t st) {
  using G = RowGeo<R>;
  CUtensorMap map{};
  if (small_tiles(n, H, W)) {
    using GS = RowGeo<R, kBHSmall>;
    dim3 grid((W + kTW - 1) / kTW, (H + kBHSmall - 1) / kBHSmall, n);
    k_dark_rows<R, false, kBHSmall><<<grid, kThreads, GS::SMEM, st>>>(in, in_fs, H, W, dark, dark_fs, frame_max,
                                                                      unit_max, map);
    return cudaGetLastError();
  }
  dim3 grid((W + kTW - 1) / kTW, (H + kBH - 1) / kBH, n);
  // the map's frame pitch must be >= one frame and the innermost extent a whole number of u64
  if (use_tma() && R <= 8 && (3LL * W) % 8 == 0 && (n == 1 || in_fs >= 3LL * W * H) &&
      make_row_map(in, n == 1 ? 3LL * W * H : in_fs, n, H, W, &map)) {
    auto kern = k_dark_rows<R, true, kBH>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM_TMA);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, G::SMEM_TMA, st>>>(in, in_fs, H, W, dark, dark_fs, frame_max, unit_max, map);
    return cudaGetLastError();
  }
  auto kern = k_dark_rows<R, false, kBH>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, G::SMEM, st>>>(in, in_fs, H, W, dark, dark_fs, frame_max, unit_max, map);
  return cudaGetLastError();
}

}  // namespace

bool dark_rows_supported(int r, int W, int64_t in_fs, int64_t dark_fs, const void* in, const void* dark) {
  return r >= 1 && r <= 16 && W % 16 == 0 && in_fs % 16 == 0 && dark_fs % 4 == 0 && (uintptr_t)in % 16 == 0 &&
         (uintptr_t)dark % 4 == 0;
}

cudaError_t dark_rows(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, uint8_t* dark,
                      int64_t dark_fs, uint32_t* frame_max, uint32_t* unit_max, cudaStream_t st) {
  switch (r) {
#define DHZ_R(k) \
  case k:        \
    return launch<k>(in, in_fs, n, H, W, dark, dark_fs, frame_max, unit_max, st);
    DHZ_R(1) DHZ_R(2) DHZ_R(3) DHZ_R(4) DHZ_R(5) DHZ_R(6) DHZ_R(7) DHZ_R(8)
    DHZ_R(9) DHZ_R(10) DHZ_R(11) DHZ_R(12) DHZ_R(13) DHZ_R(14) DHZ_R(15) DHZ_R(16)
#undef DHZ_R
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace dhz
