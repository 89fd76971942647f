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
// chain exactly, so A is bit-identical to the reference.  When K == n the
// reference takes arange(n) (:75-76).
//
// K2 (k_level_hist): K1 recorded the maximum of every 16-row x 32-column unit;
//   units below max-15 are skipped without reading (one gather tests 32 units),
//   the others count the pixels of each level in [max-15, max] per row (rare
//   shared atomics), folded into a per-row / per-frame level histogram.
// K3 (k_threshold): CTA per frame: T = K-th largest level, per-row (above,
//   tie) counts and their exclusive prefixes over rows (linear index order).
//   Frames whose top K spans more than 16 levels are redone by K3b
//   (k_full_hist / k_full_rows: a full 256-level histogram and per-row counts
//   spread over many CTAs per frame, the last CTA of each finishing the frame's
//   step; frames on the fast path exit at once).
// K4 (k_compact, k_airlight): warps compact the rows that hold selected pixels,
//   reading only the row's units whose maximum reaches T (ballot + popc, index
//   order); then a CTA per frame gathers and runs the three sequential fp64 sums.
#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

constexpr int kT = 256;
constexpr int kWarps = kT / 32;
// Row pitch of K2's warp-private (row, level) counters: odd, so the 16 rows of a unit
// (two lanes per row) counting the same level hit 16 different banks (pitch 16 put
// every other row on the same bank: 8-way conflicts on the shared atomics).
constexpr int kCntPitch = kWin + 1;

// ---------------------------------------------------------------------------
// K2: per-row level histogram of the levels [M-15, M]
// ---------------------------------------------------------------------------
// One 16 x 32 unit: count its pixels in [L, M] per (row, level) on the warp's shared
// counters, then fold them into the per-row and per-frame histograms (and re-zero).
template <bool VEC>
__device__ __forceinline__ void level_hist_unit(const uint8_t* __restrict__ dark, int64_t dark_fs, int H, int W,
                                                int f, int b, int u, uint32_t M, uint32_t* c,
                                                uint32_t* __restrict__ row_hist, uint32_t* __restrict__ frame_hist,
                                                int lane) {
  const uint32_t L = M >= (uint32_t)(kWin - 1) ? M - (kWin - 1) : 0u;
  const int y0 = b * kBandH, x0 = u * kUnitW;
  const uint8_t* base = dark + (int64_t)f * dark_fs + (int64_t)y0 * W + x0;
  if (VEC) {  // lane: row lane/2, 16 columns (W % 16 == 0: all in or all out)
    const int r = lane >> 1, x = 16 * (lane & 1);
    if (y0 + r < H && x0 + x < W) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(base + (int64_t)r * W + x));
      const uint32_t m4 = vmax4(vmax4(v.x, v.y), vmax4(v.z, v.w));
      const uint32_t mx = max(max(m4 & 0xFFu, (m4 >> 8) & 0xFFu), max((m4 >> 16) & 0xFFu, m4 >> 24));
      if (mx >= L) {
        const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const uint32_t bv = (ws[q >> 2] >> (8 * (q & 3))) & 0xFFu;
          if (bv >= L) atomicAdd(&c[r * kCntPitch + (M - bv)], 1u);
        }
      }
    }
  } else {  // lane: one column, 16 rows
    const int x = x0 + lane;
    if (x < W) {
      const int rows = min(kBandH, H - y0);
      for (int r = 0; r < rows; ++r) {
        const uint32_t bv = base[(int64_t)r * W + lane];
        if (bv >= L) atomicAdd(&c[r * kCntPitch + (M - bv)], 1u);
      }
    }
  }
  __syncwarp();
  if (lane < kWin) {  // per-level totals over the unit's rows
    uint32_t s = 0;
#pragma unroll
    for (int r = 0; r < kBandH; ++r) s += c[r * kCntPitch + lane];
    if (s) atomicAdd(frame_hist + (int64_t)f * kWin + lane, s);
  }
  __syncwarp();
  // per-row entries (a row's units are counted by different warps); rows past H hold zeros
  uint32_t* rh = row_hist + ((int64_t)f * H + y0) * kWin;
#pragma unroll
  for (int k = lane; k < kBandH * kWin; k += 32) {
    uint32_t* ck = c + (k / kWin) * kCntPitch + (k % kWin);
    const uint32_t v = *ck;
    if (v) {
      atomicAdd(rh + k, v);
      *ck = 0;
    }
  }
  __syncwarp();
}

// K2: units are dealt to warps 32 at a time, strided by the number of warps so that
// each warp's share mixes frames and bands; every lane tests one unit against its
// frame's window (one gather for 32 units) and the warp then counts the ballot's units.
template <bool VEC>
__global__ void __launch_bounds__(kT)
k_level_hist(const uint8_t* __restrict__ dark, int64_t dark_fs, int n, int H, int W,
             const uint32_t* __restrict__ frame_max, const uint32_t* __restrict__ unit_max,
             uint32_t* __restrict__ row_hist /* [n][H][16] */, uint32_t* __restrict__ frame_hist /* [n][16] */) {
  pdl_wait();  // K1 (dark map, unit maxima) complete
  __shared__ uint32_t cnt[kWarps][kBandH * kCntPitch];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nb = (H + kBandH - 1) / kBandH, nu = (W + kUnitW - 1) / kUnitW;
  const int64_t per_frame = (int64_t)nb * nu, items = (int64_t)n * per_frame;
  const int64_t nw = (int64_t)gridDim.x * kWarps;
  uint32_t* c = cnt[wid];
  for (int k = lane; k < kBandH * kCntPitch; k += 32) c[k] = 0;
  __syncwarp();
  for (int64_t base = (int64_t)blockIdx.x * kWarps + wid; base < items; base += 32 * nw) {
    const int64_t mine = base + nw * lane;
    bool want = false;
    uint32_t M = 0;
    if (mine < items) {
      M = frame_max[mine / per_frame];
      want = unit_max[mine] >= (M >= (uint32_t)(kWin - 1) ? M - (kWin - 1) : 0u);
    }
    for (uint32_t mask = __ballot_sync(0xffffffffu, want); mask; mask &= mask - 1) {
      const int src = __ffs(mask) - 1;
      const int64_t it = base + nw * src;
      const int f = (int)(it / per_frame);
      const int rem = (int)(it - (int64_t)f * per_frame);
      const int b = rem / nu;
      level_hist_unit<VEC>(dark, dark_fs, H, W, f, b, rem - b * nu, __shfl_sync(0xffffffffu, M, src), c, row_hist,
                           frame_hist, lane);
    }
  }
  pdl_trigger();  // after the work: K3 must not take K2 slots
}

// ---------------------------------------------------------------------------
// K3: threshold + per-row (above, tie) counts and exclusive prefixes
// ---------------------------------------------------------------------------
// row_info[f][y] = {above, ties, above_prefix, tie_prefix}
template <typename Get>
__device__ void scan_rows(int H, uint32_t* info, Get get) {
  __shared__ uint32_t tmp[32];
  const int cpt = (H + (int)blockDim.x - 1) / (int)blockDim.x;
  const int y0 = threadIdx.x * cpt, y1 = min(H, y0 + cpt);
  uint32_t la = 0, lt = 0;
  for (int y = y0; y < y1; ++y) {
    uint32_t a, t;
    get(y, a, t);
    la += a;
    lt += t;
  }
  uint32_t pa = block_exclusive_scan(la, tmp, nullptr);
  uint32_t pt = block_exclusive_scan(lt, tmp, nullptr);
  for (int y = y0; y < y1; ++y) {
    uint32_t a, t;
    get(y, a, t);
    reinterpret_cast<uint4*>(info)[y] = make_uint4(a, t, pa, pt);
    pa += a;
    pt += t;
  }
}

__global__ void __launch_bounds__(kT)
k_threshold(int64_t npx, int64_t K, int H, const uint32_t* __restrict__ frame_max,
            const uint32_t* __restrict__ row_hist, const uint32_t* __restrict__ frame_hist,
            FrameSel* __restrict__ sel, uint32_t* __restrict__ full_list, uint32_t* __restrict__ row_info) {
  pdl_wait();
  const int f = blockIdx.x;
  __shared__ int js_s;
  if (threadIdx.x < 32) {  // warp 0: inclusive scan of the kWin level counts from the top
    const int lane = threadIdx.x;
    const uint32_t M = frame_max[f];
    const uint64_t h = (lane < kWin && (uint32_t)lane <= M) ? frame_hist[(int64_t)f * kWin + lane] : 0u;
    uint64_t inc = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const bool hit = K < npx && lane < kWin && (uint32_t)lane <= M && inc >= (uint64_t)K;
    const uint32_t hits = __ballot_sync(0xffffffffu, hit);
    const int js = hits ? __ffs(hits) - 1 : -1;
    const uint64_t cum = __shfl_sync(0xffffffffu, inc - h, js < 0 ? 0 : js);
    if (lane == 0) {
      const uint32_t mode = K >= npx ? kSelAll : (js < 0 ? kSelFull : kSelFast);
      sel[f].mode = mode;
      if (mode == kSelFull) full_list[1 + atomicAdd(full_list, 1u)] = (uint32_t)f;
      if (mode == kSelFast) {
        sel[f].T = M - js;
        sel[f].above = (uint32_t)cum;
      }
      js_s = mode == kSelFast ? js : -1;
    }
  }
  __syncthreads();
  const int js = js_s;
  if (js < 0) return;
  const uint32_t* rh = row_hist + (int64_t)f * H * kWin;
  scan_rows(H, row_info + (int64_t)f * H * 4, [&](int y, uint32_t& a, uint32_t& t) {
    const uint4* h4 = reinterpret_cast<const uint4*>(rh + (int64_t)y * kWin);
    uint32_t h[kWin];
#pragma unroll
    for (int q = 0; q < kWin / 4; ++q) {
      const uint4 v = h4[q];
      h[4 * q] = v.x; h[4 * q + 1] = v.y; h[4 * q + 2] = v.z; h[4 * q + 3] = v.w;
    }
    uint32_t acc = 0, tie = 0;
#pragma unroll
    for (int j = 0; j < kWin; ++j) {
      acc += j < js ? h[j] : 0u;
      tie = j == js ? h[j] : tie;
    }
    a = acc;
    t = tie;
  });
}

// Fallback for frames whose top K spans more than kWin levels below the max
// (sel.mode == kSelFull, listed by K3 in full_list = {count, frames...}): a full
// 256-level histogram and per-row counts, each spread over kFullParts CTAs per
// frame.  The grid is (kFullParts, <= kFullFrames); with no listed frame every CTA
// exits after one load.
constexpr int kFullParts = 32;
constexpr int kFullFrames = 16;

// F1: 256-level histogram of the frame's dark bytes (warp-private shared copies);
// the frame's last CTA to finish (ticket) derives T and the count above it.
template <bool VEC>
__global__ void __launch_bounds__(kT)
k_full_hist(const uint8_t* __restrict__ dark, int64_t dark_fs, int64_t npx, int64_t K, FrameSel* __restrict__ sel,
            const uint32_t* __restrict__ full_list, uint32_t* __restrict__ hist256) {
  pdl_wait();
  const uint32_t count = __ldcg(full_list);
  __shared__ uint32_t h[kWarps][256];
  __shared__ bool last;
  const int wid = threadIdx.x >> 5, part = blockIdx.x;
  for (uint32_t i = blockIdx.y; i < count; i += gridDim.y) {
    const int f = (int)__ldcg(full_list + 1 + i);
    for (int k = threadIdx.x; k < kWarps * 256; k += kT) (&h[0][0])[k] = 0;
    __syncthreads();
    const uint8_t* p = dark + f * dark_fs;
    uint32_t* hw = h[wid];
    if (VEC) {
      const int64_t U = npx / 16, u0 = U * part / kFullParts, u1 = U * (part + 1) / kFullParts;
      for (int64_t u = u0 + threadIdx.x; u < u1; u += kT) {
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p) + u);
        const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 16; ++q) atomicAdd(&hw[(ws[q >> 2] >> (8 * (q & 3))) & 0xFFu], 1u);
      }
    } else {
      const int64_t q0 = npx * part / kFullParts, q1 = npx * (part + 1) / kFullParts;
      for (int64_t q = q0 + threadIdx.x; q < q1; q += kT) atomicAdd(&hw[p[q]], 1u);
    }
    __syncthreads();
    uint32_t* fh = hist256 + (int64_t)f * 256;
    for (int b = threadIdx.x; b < 256; b += kT) {
      uint32_t c = 0;
      for (int w = 0; w < kWarps; ++w) c += h[w][b];
      if (c) atomicAdd(fh + b, c);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&sel[f].ticket, 1u) == kFullParts - 1;
    __syncthreads();
    if (last && threadIdx.x == 0) {
      __threadfence();
      uint64_t cum = 0;
      int T = 0;
      for (int v = 255; v >= 0; --v) {
        const uint32_t c = __ldcg(fh + v);
        if (cum + c >= (uint64_t)K) {
          T = v;
          break;
        }
        cum += c;
      }
      sel[f].T = (uint32_t)T;
      sel[f].above = (uint32_t)cum;
    }
  }
}

// F2: per-row (above, tie) counts, warp per row, rows spread over kFullParts CTAs; the
// frame's last CTA writes the exclusive prefixes and moves the frame to the fast path.
__global__ void __launch_bounds__(kT)
k_full_rows(const uint8_t* __restrict__ dark, int64_t dark_fs, int H, int W, FrameSel* __restrict__ sel,
            const uint32_t* __restrict__ full_list, uint32_t* __restrict__ row_info) {
  pdl_wait();
  const uint32_t count = __ldcg(full_list);
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, part = blockIdx.x;
  for (uint32_t i = blockIdx.y; i < count; i += gridDim.y) {
    const int f = (int)__ldcg(full_list + 1 + i);
    const uint32_t T = __ldcg(&sel[f].T);
    const uint8_t* p = dark + f * dark_fs;
    uint4* info = reinterpret_cast<uint4*>(row_info + (int64_t)f * H * 4);
    for (int y = part * kWarps + wid; y < H; y += kWarps * kFullParts) {
      uint32_t na = 0, nt = 0;
      for (int x = lane; x < W; x += 32) {
        const uint32_t b = p[(int64_t)y * W + x];
        na += b > T;
        nt += b == T;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        na += __shfl_xor_sync(0xffffffffu, na, o);
        nt += __shfl_xor_sync(0xffffffffu, nt, o);
      }
      if (lane == 0) info[y] = make_uint4(na, nt, 0u, 0u);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&sel[f].ticket2, 1u) == kFullParts - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      scan_rows(H, row_info + (int64_t)f * H * 4, [&](int y, uint32_t& a, uint32_t& t) {
        const uint4 v = __ldcg(info + y);
        a = v.x;
        t = v.y;
      });
      __syncthreads();
      if (threadIdx.x == 0) sel[f].mode = kSelFast;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K4: ordered compaction of the rows holding selected pixels + sequential sum
// ---------------------------------------------------------------------------
// One row: only its 32-column units whose maximum reaches T can hold selected pixels.
// Lane l owns column 32u + l of each such unit, so each unit is one coalesced 32-byte
// read and its above/tie pixels are placed by ballot + popc in index order.  Up to 8
// units' loads are in flight together.
__device__ void compact_row(const uint8_t* __restrict__ row, const uint32_t* __restrict__ um, int nu, int W,
                            uint32_t base_idx, uint32_t T, uint32_t above, uint32_t need, uint32_t ao, uint32_t to,
                            uint32_t* __restrict__ out, int lane) {
  constexpr int kU = 8;
  const uint32_t lt = (1u << lane) - 1u;
  for (int u0 = 0; u0 < nu; u0 += 32) {
    const int um_i = u0 + lane;
    uint32_t hot = __ballot_sync(0xffffffffu, um_i < nu && __ldcg(um + um_i) >= T);
    while (hot) {
      int us[kU];
      int cnt = 0;
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        us[k] = hot ? u0 + __ffs(hot) - 1 : -1;
        cnt += hot != 0;
        hot &= hot - 1;
      }
      uint32_t bv[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int x = kUnitW * us[k] + lane;
        bv[k] = (us[k] >= 0 && x < W) ? (uint32_t)__ldcg(row + x) : 0u;
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        if (k >= cnt) break;  // warp-uniform
        const int x = kUnitW * us[k] + lane;
        const bool ok = x < W;
        const uint32_t am = __ballot_sync(0xffffffffu, ok && bv[k] > T);
        const uint32_t tm = __ballot_sync(0xffffffffu, ok && bv[k] == T);
        if (ok && bv[k] > T) {
          out[ao + __popc(am & lt)] = base_idx + x;
        } else if (ok && bv[k] == T) {
          const uint32_t r = to + __popc(tm & lt);
          if (r < need) out[above + r] = base_idx + x;
        }
        ao += __popc(am);
        to += __popc(tm);
      }
    }
  }
}

// The gather of chunk c+1 (warps 1..7) overlaps the sequential sums of chunk c
// (lanes 0..2 of warp 0), so large K is bound by the three dependent fp64 chains.
__device__ void airlight_sum(const uint8_t* __restrict__ frame, const uint32_t* __restrict__ idx, int64_t K,
                             bool all, double alpha, double* __restrict__ A) {
  constexpr int kChunk = 512;  // small first gather: the chains start early
  __shared__ double tab[256];
  __shared__ uint32_t buf[2][kChunk];
  for (int v = threadIdx.x; v < 256; v += kT) tab[v] = __ddiv_rn((double)v, 255.0);
  auto gather = [&](int64_t base, uint32_t* dst, int t0, int stride) {
    const int cnt = (int)min((int64_t)kChunk, K - base);
    // all of a thread's index loads first, then all of its pixel loads (two rounds of
    // memory latency per chunk instead of two per element)
    constexpr int kMaxPer = 4;  // kChunk / (kT - 32) rounded up
    int64_t px[kMaxPer];
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
      const int e = t0 + j * stride;
      px[j] = e < cnt ? (all ? base + e : (int64_t)__ldcg(idx + base + e)) : -1;
    }
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
      if (px[j] >= 0) {
        const uint8_t* q = frame + 3 * px[j];
        dst[t0 + j * stride] = (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16);
      }
    }
  };
  gather(0, buf[0], threadIdx.x, kT);
  __syncthreads();
  double acc = 0.0;
  const int sh = 8 * (threadIdx.x < 3 ? threadIdx.x : 0);
  int cur = 0;
  for (int64_t base = 0; base < K; base += kChunk, cur ^= 1) {
    const int cnt = (int)min((int64_t)kChunk, K - base);
    if (threadIdx.x >= 32) {
      if (base + kChunk < K) gather(base + kChunk, buf[cur ^ 1], threadIdx.x - 32, kT - 32);
    } else if (threadIdx.x < 3) {  // lanes 0..2 of warp 0: one sequential chain per channel
      const uint32_t* b = buf[cur];
      int e = 0;
      // unrolled: later groups' shared loads issue ahead of this group's dependent adds
#pragma unroll 4
      for (; e + 8 <= cnt; e += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = tab[(b[e + u] >> sh) & 0xFFu];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
      }
      for (; e < cnt; ++e) acc = __dadd_rn(acc, tab[(b[e] >> sh) & 0xFFu]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 3) {
    const double mean = __ddiv_rn(acc, (double)K);
    A[threadIdx.x] = fmax(__dmul_rn(alpha, mean), 1e-6);
  }
}

// Warp per row; a frame's rows are spread over kCompactParts CTAs.
constexpr int kCompactParts = 8;

__global__ void __launch_bounds__(kT)
k_compact(const uint8_t* __restrict__ dark, int64_t dark_fs, int64_t npx, int64_t K, int H, int W,
          const FrameSel* __restrict__ sel, const uint32_t* __restrict__ row_info,
          const uint32_t* __restrict__ unit_max, uint32_t* __restrict__ sel_idx) {
  pdl_wait();
  const int f = blockIdx.y, part = blockIdx.x;
  const uint32_t mode = sel[f].mode;
  uint32_t* out = sel_idx + (int64_t)f * K;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (mode == kSelAll) {  // K == n: arange(n)
    for (int64_t q = (int64_t)part * kT + threadIdx.x; q < npx; q += (int64_t)kT * kCompactParts)
      out[q] = (uint32_t)q;
    return;
  }
  const uint32_t T = sel[f].T, above = sel[f].above;
  const uint32_t need = (uint32_t)K - above;
  const uint4* info = reinterpret_cast<const uint4*>(row_info + (int64_t)f * H * 4);
  const uint8_t* p = dark + f * dark_fs;
  const int nb = (H + kBandH - 1) / kBandH, nu = (W + kUnitW - 1) / kUnitW;
  const uint32_t* fum = unit_max + (int64_t)f * nb * nu;
  // the warp's rows are y0, y0 + S, y0 + 2S, ...: each lane tests one of 32 of them,
  // then the warp compacts the rows the ballot marks, in order
  constexpr int S = kWarps * kCompactParts;
  for (int y0 = part * kWarps + wid; y0 < H; y0 += 32 * S) {
    const int ym = y0 + S * lane;
    uint4 ri = make_uint4(0u, 0u, 0u, 0u);  // above, ties, above_prefix, tie_prefix
    if (ym < H) ri = info[ym];
    const bool want = ri.x != 0 || (ri.y != 0 && ri.w < need);
    for (uint32_t mask = __ballot_sync(0xffffffffu, want); mask; mask &= mask - 1) {
      const int src = __ffs(mask) - 1;
      const int y = y0 + S * src;
      const uint32_t pa = __shfl_sync(0xffffffffu, ri.z, src), pt = __shfl_sync(0xffffffffu, ri.w, src);
      compact_row(p + (int64_t)y * W, fum + (int64_t)(y / kBandH) * nu, nu, W, (uint32_t)((int64_t)y * W), T,
                  above, need, pa, pt, out, lane);
    }
  }
}

__global__ void __launch_bounds__(kT)
k_airlight(const uint8_t* __restrict__ in, int64_t in_fs, int64_t K, double alpha, const FrameSel* __restrict__ sel,
           const uint32_t* __restrict__ sel_idx, double* __restrict__ airlight) {
  pdl_wait();
  const int f = blockIdx.x;
  airlight_sum(in + f * in_fs, sel_idx + (int64_t)f * K, K, sel[f].mode == kSelAll, alpha, airlight + 3 * f);
}

}  // namespace

size_t select_row_hist_bytes(int n, int H) { return 4ull * kWin * (size_t)n * H; }

cudaError_t select_u8(const uint8_t* dark, int64_t dark_fs, const uint8_t* in, int64_t in_fs, int n, int64_t npx,
                      int64_t K, double alpha, const SelectWs& ws, double* airlight, cudaStream_t st) {
  const int H = ws.H, W = ws.W;
  const bool vec = (W % 16 == 0) && (dark_fs % 16 == 0) && ((uintptr_t)dark % 16 == 0);
  const int nb = (H + kBandH - 1) / kBandH, nu = (W + kUnitW - 1) / kUnitW;
  const int64_t items = (int64_t)n * nb * nu;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // at least ~4 units per warp slot: a single small frame's few hundred units are spread
  // over many warps (each lane-group then holds few qualifying units; integer counts, so
  // the split never changes a result); large batches are capped at 8 CTAs per SM
  const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>((items + 4 * kWarps - 1) / (4 * kWarps), 8LL * sms));
  // every kernel of the chain is launched programmatically dependent (PDL) on the one before
  cudaError_t e;
  if ((e = launch_k(vec ? k_level_hist<true> : k_level_hist<false>, g2, kT, 0, st, true, dark, dark_fs, n, H, W,
                    (const uint32_t*)ws.frame_max, (const uint32_t*)ws.unit_max, ws.row_hist, ws.frame_hist)))
    return e;
  if ((e = launch_k(k_threshold, n, kT, 0, st, true, npx, K, H, (const uint32_t*)ws.frame_max,
                    (const uint32_t*)ws.row_hist, (const uint32_t*)ws.frame_hist, ws.sel, ws.full_list, ws.row_info)))
    return e;
  const dim3 cgrid(kCompactParts, n), fgrid(kFullParts, std::min(n, kFullFrames));
  if ((e = launch_k(vec ? k_full_hist<true> : k_full_hist<false>, fgrid, kT, 0, st, true, dark, dark_fs, npx, K,
                    ws.sel, (const uint32_t*)ws.full_list, ws.hist256)))
    return e;
  if ((e = launch_k(k_full_rows, fgrid, kT, 0, st, true, dark, dark_fs, H, W, ws.sel, (const uint32_t*)ws.full_list,
                    ws.row_info)))
    return e;
  if ((e = launch_k(k_compact, cgrid, kT, 0, st, true, dark, dark_fs, npx, K, H, W, (const FrameSel*)ws.sel,
                    (const uint32_t*)ws.row_info, (const uint32_t*)ws.unit_max, ws.sel_idx)))
    return e;
  if ((e = launch_k(k_airlight, n, kT, 0, st, true, in, in_fs, K, alpha, (const FrameSel*)ws.sel,
                    (const uint32_t*)ws.sel_idx, airlight)))
    return e;
  return cudaGetLastError();
}

}  // namespace dhz
