// K2..K4 — ordered top-K airlight selection on the u8 dark map and the exact
// sequential fp64 airlight mean.
//
// Reference: estimation.py:46-84 (estimate_airlight).
//   K = max(1, floor(top_fraction * n))                      (:72, computed on the host)
//   T = K-th largest dark value                              (:79, np.partition)
//   selected = [i : d_i > T] ++ first (K - above) of [i : d_i == T]   (:80-82)
//   A = max(alpha * mean(RGB[selected], axis=0), 1e-6)       (:83-84)
// numpy's axis-0 mean of a (K, 3) array is a sequential row accumulation in
// the selection order followed by a true division by K; K4 reproduces that
// chain exactly, so A is bit-identical to the reference.
//
// K2 (k_window_hist): per 16 KB segment of a frame's dark map, a 16-bin
//   histogram of the levels [max-15, max] (max from K1).  Only words with a
//   byte >= max-15 touch shared memory, so the pass is a pure 1 B/px stream.
//   The last segment-block of each frame (threadfence + ticket) finds T and
//   writes per-segment (above, tie) counts and their exclusive prefixes.
// K2b (k_full_hist): fallback when the top K pixels span more than 16 levels
//   below the max (or the frame is degenerate): full 256-bin histograms.
// K3 (k_compact): blocks whose segment holds selected pixels write their flat
//   indices, in index order, at the prefix offsets.
// K4 (k_airlight_sum): one warp per frame gathers the K selected pixels and
//   lanes 0..2 run the per-channel sequential fp64 sums.
#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

constexpr int kT = 256;  // threads per select block

__device__ __forceinline__ uint32_t ldcg_u32(const uint32_t* p) { return __ldcg(p); }

// Exclusive scan over S segments of two counters produced by `get(s, &a, &t)`;
// writes meta[s] = {a, t, a_prefix, t_prefix}.  Called by a whole block.
template <typename Get>
__device__ void scan_segments(int S, uint32_t* meta, Get get) {
  __shared__ uint32_t tmp[32];
  const int cpt = (S + kT - 1) / kT;
  const int s0 = threadIdx.x * cpt;
  uint32_t la = 0, lt = 0;
  for (int s = s0; s < min(S, s0 + cpt); ++s) {
    uint32_t a, t;
    get(s, a, t);
    la += a;
    lt += t;
  }
  uint32_t ta, tt;
  uint32_t pa = block_exclusive_scan(la, tmp, &ta);
  uint32_t pt = block_exclusive_scan(lt, tmp, &tt);
  for (int s = s0; s < min(S, s0 + cpt); ++s) {
    uint32_t a, t;
    get(s, a, t);
    meta[4 * s + 0] = a;
    meta[4 * s + 1] = t;
    meta[4 * s + 2] = pa;
    meta[4 * s + 3] = pt;
    pa += a;
    pt += t;
  }
}

__device__ __forceinline__ bool last_block_of_frame(uint32_t* ticket, int S) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t t = atomicAdd(ticket, 1u);
    is_last = (t == (uint32_t)S - 1u);
    if (is_last) *ticket = 0u;  // every other block of the frame has arrived
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}

template <bool VEC>
__global__ void __launch_bounds__(kT)
k_window_hist(const uint8_t* __restrict__ dark, int64_t dark_fs, int64_t npx, int64_t K, int S, int W,
              const uint32_t* __restrict__ frame_max, const uint32_t* __restrict__ band_max,
              FrameSel* __restrict__ sel, uint32_t* __restrict__ seg_hist, uint32_t* __restrict__ seg_meta) {
  __shared__ uint32_t h[kWin];
  const int f = blockIdx.y, s = blockIdx.x;
  if (threadIdx.x < kWin) h[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t M = frame_max[f];
  const uint32_t L = M >= (uint32_t)(kWin - 1) ? M - (kWin - 1) : 0u;
  const uint32_t Mw = M * 0x01010101u, Lw = L * 0x01010101u;
  const int64_t b0 = (int64_t)s * kSeg;
  const int64_t b1 = min(npx, b0 + kSeg);
  const uint8_t* p = dark + f * dark_fs;
  // Skip the read when no 16-row band touching this segment reaches the window
  // (K1's band maxima): most segments of a natural frame.
  bool hot = false;
  {
    const int64_t H = npx / W, nb = (H + 15) / 16;
    const int64_t blo = (b0 / W) / 16, bhi = ((b1 - 1) / W) / 16;
    for (int64_t bb = blo + threadIdx.x; bb <= bhi; bb += kT) hot |= band_max[f * nb + bb] >= L;
  }
  if (__syncthreads_or(hot)) {
  uint32_t c0 = 0;
  auto word = [&](uint32_t w) {
    if (w == Mw) {
      c0 += 4;
    } else if (__vcmpgeu4(w, Lw)) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t b = (w >> (8 * k)) & 0xFFu;
        if (b >= L) atomicAdd(&h[M - b], 1u);
      }
    }
  };
  auto byte = [&](uint32_t b) {
    if (b == M) c0 += 1;
    else if (b >= L) atomicAdd(&h[M - b], 1u);
  };
  if (VEC) {
#pragma unroll
    for (int j = 0; j < kSeg / (16 * kT); ++j) {
      const int64_t off = b0 + 16 * (j * kT + threadIdx.x);
      if (off + 16 <= b1) {
        const uint4 v = ldg_nc_v4(p + off);
        // max of the 16 bytes on 16-bit lanes (native VIMNMX3), then the rare
        // per-word pass only when some byte reaches the window
        const uint32_t mx = max3u(max3u(unpack_lo(v.x), unpack_hi(v.x), unpack_lo(v.y)),
                                  max3u(unpack_hi(v.y), unpack_lo(v.z), unpack_hi(v.z)),
                                  max2(unpack_lo(v.w), unpack_hi(v.w)));
        if (max(mx & 0xFFFFu, mx >> 16) >= L) {
          word(v.x); word(v.y); word(v.z); word(v.w);
        }
      } else {
        for (int64_t q = off; q < b1 && q < off + 16; ++q) byte(p[q]);
      }
    }
  } else {
    for (int64_t q = b0 + threadIdx.x; q < b1; q += kT) byte(p[q]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c0 += __shfl_xor_sync(0xffffffffu, c0, o);
  if ((threadIdx.x & 31) == 0 && c0) atomicAdd(&h[0], c0);
  }
  __syncthreads();
  uint32_t* mine = seg_hist + ((int64_t)f * S + s) * kWin;
  if (threadIdx.x < kWin) mine[threadIdx.x] = h[threadIdx.x];

  if (!last_block_of_frame(&sel[f].ticket, S)) return;

  // ---- last block of frame f: threshold and per-segment prefix offsets ----
  __shared__ uint32_t part[kT / kWin][kWin];
  __shared__ uint32_t tot[kWin];
  __shared__ int jstar_s;
  const uint32_t* fh = seg_hist + (int64_t)f * S * kWin;
  {
    const int j = threadIdx.x % kWin, pi = threadIdx.x / kWin;
    uint32_t acc = 0;
    for (int ss = pi; ss < S; ss += kT / kWin) acc += ldcg_u32(fh + ss * kWin + j);
    part[pi][j] = acc;
  }
  __syncthreads();
  if (threadIdx.x < kWin) {
    uint32_t acc = 0;
    for (int i = 0; i < kT / kWin; ++i) acc += part[i][threadIdx.x];
    tot[threadIdx.x] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int js = -1;
    uint32_t mode = kSelFast, above = 0;
    if (K >= npx) {
      mode = kSelAll;
    } else {
      uint64_t cum = 0;
      for (int j = 0; j < kWin && (uint32_t)j <= M; ++j) {
        if (cum + tot[j] >= (uint64_t)K) { js = j; break; }
        cum += tot[j];
      }
      if (js < 0) {
        mode = kSelFull;
      } else {
        above = (uint32_t)cum;
        sel[f].T = M - js;
        sel[f].above = above;
      }
    }
    sel[f].mode = mode;
    jstar_s = (mode == kSelFast) ? js : -1;
  }
  __syncthreads();
  const int js = jstar_s;
  if (js < 0) return;
  scan_segments(S, seg_meta + (int64_t)f * S * 4, [&](int ss, uint32_t& a, uint32_t& t) {
    const uint32_t* hh = fh + ss * kWin;
    uint32_t acc = 0;
    for (int j = 0; j < js; ++j) acc += ldcg_u32(hh + j);
    a = acc;
    t = ldcg_u32(hh + js);
  });
}

template <bool VEC>
__global__ void __launch_bounds__(kT)
k_full_hist(const uint8_t* __restrict__ dark, int64_t dark_fs, int64_t npx, int64_t K, int S,
            FrameSel* __restrict__ sel, uint32_t* __restrict__ seg_full, uint32_t* __restrict__ seg_meta) {
  const int f = blockIdx.y, s = blockIdx.x;
  if (sel[f].mode != kSelFull) return;  // uniform per frame: all blocks of f agree
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t b0 = (int64_t)s * kSeg;
  const int64_t b1 = min(npx, b0 + kSeg);
  const uint8_t* p = dark + f * dark_fs;
  for (int64_t q = b0 + threadIdx.x; q < b1; q += kT) atomicAdd(&h[p[q]], 1u);
  __syncthreads();
  uint32_t* mine = seg_full + ((int64_t)f * S + s) * 256;
  mine[threadIdx.x] = h[threadIdx.x];

  if (!last_block_of_frame(&sel[f].ticket2, S)) return;

  const uint32_t* fh = seg_full + (int64_t)f * S * 256;
  __shared__ uint32_t tot[256];
  __shared__ int T_s;
  {
    uint32_t acc = 0;
    for (int ss = 0; ss < S; ++ss) acc += ldcg_u32(fh + ss * 256 + threadIdx.x);
    tot[threadIdx.x] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t cum = 0;
    int T = 0;
    for (int v = 255; v >= 0; --v) {
      if (cum + tot[v] >= (uint64_t)K) { T = v; break; }
      cum += tot[v];
    }
    sel[f].T = (uint32_t)T;
    sel[f].above = (uint32_t)cum;
    T_s = T;
  }
  __syncthreads();
  const int T = T_s;
  scan_segments(S, seg_meta + (int64_t)f * S * 4, [&](int ss, uint32_t& a, uint32_t& t) {
    const uint32_t* hh = fh + ss * 256;
    uint32_t acc = 0;
    for (int v = T + 1; v < 256; ++v) acc += ldcg_u32(hh + v);
    a = acc;
    t = ldcg_u32(hh + T);
  });
  __syncthreads();
  if (threadIdx.x == 0) sel[f].mode = kSelFast;
}

template <bool VEC>
__global__ void __launch_bounds__(kT)
k_compact(const uint8_t* __restrict__ dark, int64_t dark_fs, int64_t npx, int64_t K, int S,
          const FrameSel* __restrict__ sel, const uint32_t* __restrict__ seg_meta,
          uint32_t* __restrict__ sel_idx) {
  const int f = blockIdx.y, s = blockIdx.x;
  const uint32_t mode = sel[f].mode;
  if (mode == kSelAll) {  // K == n: the reference takes arange(n) (estimation.py:75-76)
    uint32_t* out = sel_idx + (int64_t)f * K;
    for (int64_t q = (int64_t)s * kSeg + threadIdx.x; q < min(npx, (int64_t)(s + 1) * kSeg); q += kT)
      out[q] = (uint32_t)q;
    return;
  }
  if (mode != kSelFast) return;
  const uint32_t T = sel[f].T, above = sel[f].above;
  const uint32_t need = (uint32_t)K - above;
  const uint32_t* mt = seg_meta + ((int64_t)f * S + s) * 4;
  const uint32_t na_s = mt[0], nt_s = mt[1], ao = mt[2], to = mt[3];
  if (na_s == 0 && (nt_s == 0 || to >= need)) return;
  const int64_t b0 = (int64_t)s * kSeg + 64 * threadIdx.x;
  const int64_t b1 = min(npx, (int64_t)s * kSeg + kSeg);
  const uint8_t* p = dark + f * dark_fs;
  uint32_t w[16];
  if (VEC && b0 + 64 <= b1) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 v = ldg_nc_v4(p + b0 + 16 * j);
      w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      uint32_t word = 0;
      for (int k = 0; k < 4; ++k) {
        const int64_t q = b0 + 4 * j + k;
        // bytes past the frame end can never be selected: give them 0 and a
        // level strictly below T by masking below.
        const uint32_t b = (q < b1) ? p[q] : 0u;
        word |= b << (8 * k);
      }
      w[j] = word;
    }
  }
  const int nvalid = (int)max((int64_t)0, min((int64_t)64, b1 - b0));
  uint32_t na = 0, nt = 0;
  for (int k = 0; k < nvalid; ++k) {
    const uint32_t b = (w[k >> 2] >> (8 * (k & 3))) & 0xFFu;
    na += (b > T);
    nt += (b == T);
  }
  __shared__ uint32_t tmp[32];
  uint32_t pa = block_exclusive_scan(na, tmp, nullptr);
  uint32_t pt = block_exclusive_scan(nt, tmp, nullptr);
  if (na == 0 && nt == 0) return;
  uint32_t* out = sel_idx + (int64_t)f * K;
  const uint32_t base_idx = (uint32_t)b0;
  for (int k = 0; k < nvalid; ++k) {
    const uint32_t b = (w[k >> 2] >> (8 * (k & 3))) & 0xFFu;
    if (b > T) {
      out[ao + pa++] = base_idx + k;
    } else if (b == T) {
      const uint32_t r = to + pt++;
      if (r < need) out[above + r] = base_idx + k;
    }
  }
}

constexpr int kSumWarps = 4;
constexpr int kChunk = 256;

__global__ void __launch_bounds__(32 * kSumWarps)
k_airlight_sum(const uint8_t* __restrict__ in, int64_t in_fs, int n, int64_t npx, int64_t K, double alpha,
               const FrameSel* __restrict__ sel, const uint32_t* __restrict__ sel_idx,
               double* __restrict__ airlight) {
  __shared__ double tab[256];
  __shared__ uint32_t buf[kSumWarps][kChunk];
  for (int v = threadIdx.x; v < 256; v += blockDim.x) tab[v] = __ddiv_rn((double)v, 255.0);
  __syncthreads();
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x * kSumWarps + wid;
  if (f >= n) return;
  const bool all = sel[f].mode == kSelAll;
  const uint8_t* frame = in + f * in_fs;
  const uint32_t* idx = sel_idx + (int64_t)f * K;
  double acc = 0.0;
  const int sh = 8 * (lane < 3 ? lane : 0);
  for (int64_t base = 0; base < K; base += kChunk) {
    const int cnt = (int)min((int64_t)kChunk, K - base);
    for (int e = lane; e < cnt; e += 32) {
      const int64_t px = all ? base + e : (int64_t)idx[base + e];
      const uint8_t* q = frame + 3 * px;
      buf[wid][e] = (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16);
    }
    __syncwarp();
    if (lane < 3) {
      int e = 0;
      for (; e + 8 <= cnt; e += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = tab[(buf[wid][e + u] >> sh) & 0xFFu];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
      }
      for (; e < cnt; ++e) acc = __dadd_rn(acc, tab[(buf[wid][e] >> sh) & 0xFFu]);
    }
    __syncwarp();
  }
  if (lane < 3) {
    const double mean = __ddiv_rn(acc, (double)K);
    airlight[3 * f + lane] = fmax(__dmul_rn(alpha, mean), 1e-6);
  }
}

}  // namespace

cudaError_t select_u8(const uint8_t* dark, int64_t dark_fs, int n, int64_t npx, int64_t K,
                      const SelectWs& ws, cudaStream_t st) {
  const bool vec = (npx % 16 == 0) && (dark_fs % 16 == 0) && ((uintptr_t)dark % 16 == 0);
  dim3 grid(ws.S, n);
  if (vec) {
    k_window_hist<true><<<grid, kT, 0, st>>>(dark, dark_fs, npx, K, ws.S, ws.W, ws.frame_max, ws.band_max,
                                              ws.sel, ws.seg_hist, ws.seg_meta);
    k_full_hist<true><<<grid, kT, 0, st>>>(dark, dark_fs, npx, K, ws.S, ws.sel, ws.seg_full, ws.seg_meta);
    k_compact<true><<<grid, kT, 0, st>>>(dark, dark_fs, npx, K, ws.S, ws.sel, ws.seg_meta, ws.sel_idx);
  } else {
    k_window_hist<false><<<grid, kT, 0, st>>>(dark, dark_fs, npx, K, ws.S, ws.W, ws.frame_max, ws.band_max,
                                               ws.sel, ws.seg_hist, ws.seg_meta);
    k_full_hist<false><<<grid, kT, 0, st>>>(dark, dark_fs, npx, K, ws.S, ws.sel, ws.seg_full, ws.seg_meta);
    k_compact<false><<<grid, kT, 0, st>>>(dark, dark_fs, npx, K, ws.S, ws.sel, ws.seg_meta, ws.sel_idx);
  }
  return cudaGetLastError();
}

cudaError_t airlight_sum_u8(const uint8_t* in, int64_t in_fs, int n, int64_t npx, int64_t K, double alpha,
                            const SelectWs& ws, double* airlight, cudaStream_t st) {
  const int blocks = (n + kSumWarps - 1) / kSumWarps;
  k_airlight_sum<<<blocks, 32 * kSumWarps, 0, st>>>(in, in_fs, n, npx, K, alpha, ws.sel, ws.sel_idx, airlight);
  return cudaGetLastError();
}

}  // namespace dhz
