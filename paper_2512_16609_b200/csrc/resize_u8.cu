// Default video mode (the reference's DehazeParams() resizes every frame to
// resize_to = (640, 480)): pixel-centre bilinear resize in float64
// (imageops.py:47-78) followed by the video pipeline at the working size
// (pipeline.py:175-215), batched over frames.
//
// After the resize the image is no longer on the 1/255 grid, so the u8 LUT path
// does not apply; everything here is float64 with the reference's rounding
// order.  The resized image is never stored: the dark pass and the recovery
// pass recompute it from the u8 input (four source pixels per sample, read
// through L1/L2), which is cheaper than writing and re-reading 24 B/px.
//
//   R1 k_rs_dark     32x64 output tile + halo: resized channel minimum, separable
//                    erosion in shared memory (exact selection), dark map (fp64)
//                    and a per-frame histogram of floor(dark * 4096).
//   R2 k_rs_select   one CTA per frame: the bucket holding the K-th largest value,
//                    ordered compaction of the candidates (bucket >= B) into shared
//                    memory, radix select of the exact K-th largest value T among
//                    them, the reference's tie rule (values > T in index order, then
//                    the first K-above ties, estimation.py:71-82) and the sequential
//                    fp64 airlight sum (:83-84).  A frame with more candidates than
//                    fit runs the same steps over its whole dark map.
//   R3 k_rs_recover  per output pixel: resized RGB, channel minimum, coarse t
//                    (estimation.py:100-101), recovery (recover.py:40-43) and the
//                    output byte from the exact thresholds of gamma + float_to_u8;
//                    with gray-world balance a sums pass, per-frame thresholds
//                    (balance_thresholds) and a bytes pass.
#include <algorithm>

#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

constexpr int kTH = 32, kTW = 64;   // R1 output tile
constexpr int kT1 = 256;            // R1 threads
constexpr int kT2 = 512;            // R2 threads (4 CTAs/SM: a 300-frame batch is one wave; 1024 ran it as 148 + 148 + 4)
constexpr int kCap = 4096;          // R2 candidates kept in shared memory
constexpr int kT3 = 256;            // R3 threads
constexpr int kColTab = 1024;       // R3: output widths up to this use a column-tap table

__device__ __forceinline__ double u8f(uint32_t v) { return __ddiv_rn((double)v, 255.0); }

// Source sample of output coordinate i (imageops.py:64-72): clip((i + 0.5) * scale - 0.5, 0, n - 1).
struct Tap {
  int i0, i1;
  double f, g;  // weight of i1 and of i0 (1 - f)
};
__device__ __forceinline__ Tap tap(int i, double scale, int n) {
  double s = __dsub_rn(__dmul_rn(__dadd_rn((double)i, 0.5), scale), 0.5);
  s = dmin(dmax(s, 0.0), (double)n - 1.0);
  Tap t;
  t.i0 = (int)floor(s);
  t.i1 = min(t.i0 + 1, n - 1);
  t.f = __dsub_rn(s, (double)t.i0);
  t.g = __dsub_rn(1.0, t.f);
  return t;
}

// Compact column/row tap for shared-memory tables: i1 = min(i0 + 1, n - 1) and
// g = 1 - f are recomputed (one op each) from (i0, f).
struct TapS {
  int i0;
  double f;
};
__device__ __forceinline__ Tap expand(const TapS& c, int n) {
  Tap t;
  t.i0 = c.i0;
  t.i1 = min(c.i0 + 1, n - 1);
  t.f = c.f;
  t.g = __dsub_rn(1.0, c.f);
  return t;
}
__device__ __forceinline__ TapS compact(const Tap& t) { return TapS{t.i0, t.f}; }

// Resized RGB from its row and column taps: rows blend first, then columns, clip
// (imageops.py:74-78).  Every term is >= 0, so the clip reduces to min(., 1).
__device__ __forceinline__ void resized_rgb_t(const uint8_t* __restrict__ frame, int w, const Tap& ty,
                                              const Tap& tx, const double* __restrict__ s_f, double (&rgb)[3]) {
  const uint8_t* p00 = frame + ((int64_t)ty.i0 * w + tx.i0) * 3;
  const uint8_t* p10 = frame + ((int64_t)ty.i1 * w + tx.i0) * 3;
  // A zero weight makes a blend exact: RN(RN(a*1) + RN(b*0)) == a for a >= 0 (integer
  // scale factors, e.g. 1920 -> 640, hit this on every column), so that tap is skipped.
  if (tx.f == 0.0) {
    if (ty.f == 0.0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) rgb[c] = s_f[p00[c]];
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        rgb[c] = dmin(__dadd_rn(__dmul_rn(s_f[p00[c]], ty.g), __dmul_rn(s_f[p10[c]], ty.f)), 1.0);
    }
    return;
  }
  const uint8_t* p01 = frame + ((int64_t)ty.i0 * w + tx.i1) * 3;
  const uint8_t* p11 = frame + ((int64_t)ty.i1 * w + tx.i1) * 3;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double r0 = __dadd_rn(__dmul_rn(s_f[p00[c]], ty.g), __dmul_rn(s_f[p10[c]], ty.f));
    const double r1 = __dadd_rn(__dmul_rn(s_f[p01[c]], ty.g), __dmul_rn(s_f[p11[c]], ty.f));
    rgb[c] = dmin(__dadd_rn(__dmul_rn(r0, tx.g), __dmul_rn(r1, tx.f)), 1.0);
  }
}

__device__ __forceinline__ void resized_rgb(const uint8_t* __restrict__ frame, const ResizeGeo& G, int y, int x,
                                            const double* __restrict__ s_f, double (&rgb)[3]) {
  resized_rgb_t(frame, G.w, tap(y, G.sy, G.h), tap(x, G.sx, G.w), s_f, rgb);
}

// Tap with precomputed byte offsets (row: i * 3w, column: 3 i) and both weights.
struct OffTap {
  int o0, o1;
  double f, g;
};
__device__ __forceinline__ OffTap off_tap(const Tap& t, int unit) { return OffTap{t.i0 * unit, t.i1 * unit, t.f, t.g}; }

// resized_rgb_t from offset taps (same arithmetic, same zero-weight shortcuts).
__device__ __forceinline__ void resized_rgb_o(const uint8_t* __restrict__ frame, const OffTap& ty, const OffTap& tx,
                                              const double* __restrict__ s_f, double (&rgb)[3]) {
  const uint8_t* p00 = frame + ty.o0 + tx.o0;
  const uint8_t* p10 = frame + ty.o1 + tx.o0;
  if (tx.f == 0.0) {
    if (ty.f == 0.0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) rgb[c] = s_f[p00[c]];
    } else {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        rgb[c] = dmin(__dadd_rn(__dmul_rn(s_f[p00[c]], ty.g), __dmul_rn(s_f[p10[c]], ty.f)), 1.0);
    }
    return;
  }
  const uint8_t* p01 = frame + ty.o0 + tx.o1;
  const uint8_t* p11 = frame + ty.o1 + tx.o1;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double r0 = __dadd_rn(__dmul_rn(s_f[p00[c]], ty.g), __dmul_rn(s_f[p10[c]], ty.f));
    const double r1 = __dadd_rn(__dmul_rn(s_f[p01[c]], ty.g), __dmul_rn(s_f[p11[c]], ty.f));
    rgb[c] = dmin(__dadd_rn(__dmul_rn(r0, tx.g), __dmul_rn(r1, tx.f)), 1.0);
  }
}

__device__ __forceinline__ int bucket_of(double d) { return min(max((int)(d * 4096.0), 0), kResizeBuckets - 1); }

// ------------------------------------------------------------------- R1 ----
// Sliding minimum of width 2R+1 over S outputs from S+2R inputs in registers:
// doubling (widths 2, 4, 8, 16, ...) then one combine, ~log2(2R+1)+1 fmin per output.
template <int R, int S>
__device__ __forceinline__ void window_min(const double (&v)[S + 2 * R], double (&o)[S]) {
  constexpr int L = 2 * R + 1;
  constexpr int P = L >= 32 ? 32 : L >= 16 ? 16 : L >= 8 ? 8 : L >= 4 ? 4 : L >= 2 ? 2 : 1;  // largest power <= L
  constexpr int N = S + 2 * R;
  double m[N];
#pragma unroll
  for (int i = 0; i < N; ++i) m[i] = v[i];
#pragma unroll
  for (int w = 1; w < P; w <<= 1) {
#pragma unroll
    for (int i = 0; i + w < N; ++i) m[i] = dmin(m[i], m[i + w]);
  }
  // m[i] = min over [i, i + P); the window [i, i + L) = [i, i + P) u [i + L - P, i + L)
#pragma unroll
  for (int i = 0; i < S; ++i) o[i] = dmin(m[i], m[i + L - P]);
}

// Tile kernel with the erosion radius fixed at compile time (register windows).
template <int R>
__global__ void __launch_bounds__(kT1, R <= 7 ? 4 : 2)
k_rs_dark_t(const uint8_t* __restrict__ in, int64_t in_fs, ResizeGeo G, double* __restrict__ dark,
            uint32_t* __restrict__ hist) {
  constexpr int S = 8;                       // outputs per thread and pass
  constexpr int PH = kTH + 2 * R, PW = kTW + 2 * R;
  // shared-memory pitches (in doubles): odd, so the 32 rows a warp reads in the row
  // pass (and writes as row minima) fall on 16 distinct 8-byte bank pairs
  constexpr int PWP = PW | 1, RP = kTW + 1;
  constexpr int kRowItems = PH * (kTW / S);
  constexpr int kRowIter = (kRowItems + kT1 - 1) / kT1;
  constexpr int kHistWords = (kResizeBuckets + 1) / 2;  // 16-bit counters (a tile has <= 2048 outputs)
  extern __shared__ double sm[];
  __shared__ double s_f[256];
  __shared__ uint32_t s_hist[kHistWords];
  const int f = blockIdx.z;
  const int ty0 = blockIdx.y * kTH, tx0 = blockIdx.x * kTW;
  double* cm = sm;  // [PH][PWP] resized channel minimum (clamped coordinates); then [PH][RP] row minima
  // tap tables: byte offsets of the two source rows / columns and their weights
  __shared__ OffTap s_ty[PH], s_tx[PW];
  s_f[threadIdx.x] = u8f(threadIdx.x);
  for (int b = threadIdx.x; b < kHistWords; b += kT1) s_hist[b] = 0;
  for (int k = threadIdx.x; k < PH + PW; k += kT1) {
    if (k < PH) s_ty[k] = off_tap(tap(min(max(ty0 - R + k, 0), G.H - 1), G.sy, G.h), 3 * G.w);
    else s_tx[k - PH] = off_tap(tap(min(max(tx0 - R + k - PH, 0), G.W - 1), G.sx, G.w), 3);
  }
  __syncthreads();
  const uint8_t* frame = in + (int64_t)f * in_fs;
  // a thread keeps one tile column (its column tap in registers) and walks the rows, two
  // at a time so both samples' byte loads are in flight together
  {
    constexpr int NRG = kT1 / PW;  // row groups
    const int px = threadIdx.x % PW, pr = threadIdx.x / PW;
    if (pr < NRG) {
      const OffTap cx = s_tx[px];
      for (int py = pr; py < PH; py += 2 * NRG) {
        const int py2 = min(py + NRG, PH - 1);
        double rgb[3], rgb2[3];
        resized_rgb_o(frame, s_ty[py], cx, s_f, rgb);
        resized_rgb_o(frame, s_ty[py2], cx, s_f, rgb2);
        cm[py * PWP + px] = dmin(dmin(rgb[0], rgb[1]), rgb[2]);  // estimation.py:38
        cm[py2 * PWP + px] = dmin(dmin(rgb2[0], rgb2[1]), rgb2[2]);
      }
    }
  }
  __syncthreads();
  // rows first (morphology.py:73): item = (8-column segment, row), lanes on consecutive
  // rows; all of a thread's windows are reduced into registers before the row minima
  // overwrite cm in place
  {
    double o[kRowIter][S];
#pragma unroll
    for (int k = 0; k < kRowIter; ++k) {
      const int e = threadIdx.x + k * kT1;
      if (e < kRowItems) {
        const int seg = e / PH, py = e - seg * PH;
        const double* row = cm + py * PWP + seg * S;
        double v[S + 2 * R];
#pragma unroll
        for (int i = 0; i < S + 2 * R; ++i) v[i] = row[i];
        window_min<R, S>(v, o[k]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRowIter; ++k) {
      const int e = threadIdx.x + k * kT1;
      if (e < kRowItems) {
        const int seg = e / PH, py = e - seg * PH;
#pragma unroll
        for (int i = 0; i < S; ++i) cm[py * RP + seg * S + i] = o[k][i];
      }
    }
  }
  __syncthreads();
  const double* rm = cm;  // [PH][RP]
  // columns: item = (column, 8-row segment); lanes take consecutive columns
  const int64_t npx = (int64_t)G.H * G.W;
  for (int e = threadIdx.x; e < kTW * (kTH / S); e += kT1) {
    const int seg = e / kTW, px = e - seg * kTW;
    const double* col = rm + seg * S * RP + px;
    double v[S + 2 * R], o[S];
#pragma unroll
    for (int i = 0; i < S + 2 * R; ++i) v[i] = col[i * RP];
    window_min<R, S>(v, o);
    const int x = tx0 + px;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const int y = ty0 + seg * S + i;
      if (y < G.H && x < G.W) {
        dark[(int64_t)f * npx + (int64_t)y * G.W + x] = o[i];
        const int b = bucket_of(o[i]);
        atomicAdd(&s_hist[b >> 1], 1u << (16 * (b & 1)));
      }
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < kHistWords; w += kT1) {
    const uint32_t c2 = s_hist[w];
    if (c2 & 0xFFFFu) atomicAdd(&hist[(int64_t)f * kResizeBuckets + 2 * w], c2 & 0xFFFFu);
    if (c2 >> 16) atomicAdd(&hist[(int64_t)f * kResizeBuckets + 2 * w + 1], c2 >> 16);
  }
}

// Generic radius (runtime r, loops over the window in shared memory).
__global__ void __launch_bounds__(kT1)
k_rs_dark(const uint8_t* __restrict__ in, int64_t in_fs, ResizeGeo G, int r, double* __restrict__ dark,
          uint32_t* __restrict__ hist) {
  extern __shared__ double sm[];
  __shared__ double s_f[256];
  __shared__ uint32_t s_hist[kResizeBuckets];
  const int f = blockIdx.z;
  const int ty0 = blockIdx.y * kTH, tx0 = blockIdx.x * kTW;
  const int PH = kTH + 2 * r, PW = kTW + 2 * r;
  double* cm = sm;              // [PH][PW] resized channel minimum (clamped coordinates)
  double* rm = sm + PH * PW;    // [PH][kTW] row minima
  s_f[threadIdx.x] = u8f(threadIdx.x);
  for (int b = threadIdx.x; b < kResizeBuckets; b += kT1) s_hist[b] = 0;
  __syncthreads();
  const uint8_t* frame = in + (int64_t)f * in_fs;
  for (int e = threadIdx.x; e < PH * PW; e += kT1) {
    const int py = e / PW, px = e - py * PW;
    const int y = min(max(ty0 - r + py, 0), G.H - 1), x = min(max(tx0 - r + px, 0), G.W - 1);
    double rgb[3];
    resized_rgb(frame, G, y, x, s_f, rgb);
    cm[e] = dmin(dmin(rgb[0], rgb[1]), rgb[2]);  // estimation.py:38
  }
  __syncthreads();
  for (int e = threadIdx.x; e < PH * kTW; e += kT1) {  // morphology.py:73: rows first
    const int py = e / kTW, px = e - py * kTW;
    const double* row = cm + py * PW + px;
    double v = row[0];
    for (int k = 1; k <= 2 * r; ++k) v = dmin(v, row[k]);
    rm[e] = v;
  }
  __syncthreads();
  const int64_t npx = (int64_t)G.H * G.W;
  for (int e = threadIdx.x; e < kTH * kTW; e += kT1) {
    const int py = e / kTW, px = e - py * kTW;
    const int y = ty0 + py, x = tx0 + px;
    if (y < G.H && x < G.W) {
      const double* col = rm + py * kTW + px;
      double v = col[0];
      for (int k = 1; k <= 2 * r; ++k) v = dmin(v, col[k * kTW]);
      dark[(int64_t)f * npx + (int64_t)y * G.W + x] = v;
      atomicAdd(&s_hist[bucket_of(v)], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kResizeBuckets; b += kT1)
    if (s_hist[b]) atomicAdd(&hist[(int64_t)f * kResizeBuckets + b], s_hist[b]);
}

// ------------------------------------------------------------------- R2 ----
// Order-preserving key of a non-negative double (-0.0 reads as +0.0).
__device__ __forceinline__ uint64_t key_of(double d) {
  return (uint64_t)__double_as_longlong(d == 0.0 ? 0.0 : d) | 0x8000000000000000ull;
}

struct SelShared {
  uint32_t hist[256];
  uint32_t scan_tmp[32];
  uint64_t prefix;
  long long krem;
  uint32_t total;
};

// K-th largest key among values get(j), j < m (radix select, 8 passes of 8 bits).
template <class Get>
__device__ uint64_t radix_kth(const Get& get, int64_t m, int64_t K, SelShared& S) {
  if (threadIdx.x == 0) {
    S.prefix = 0;
    S.krem = K;
  }
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) S.hist[b] = 0;
    __syncthreads();
    const uint64_t prefix = S.prefix;
    const uint64_t pmask = pass == 0 ? 0ull : (~0ull << (64 - 8 * pass));
    for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
      const uint64_t k = key_of(get(j));
      if ((k & pmask) == prefix) atomicAdd(&S.hist[(k >> shift) & 0xFFu], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // warp 0: digit holding the krem-th largest
      const int lane = threadIdx.x;
      uint32_t c[8], s = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // lane owns digits 255-8*lane .. 248-8*lane (descending)
        c[u] = S.hist[255 - 8 * lane - u];
        s += c[u];
      }
      uint32_t inc = s;  // inclusive prefix over lanes (descending digit order)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const long long krem = S.krem;
      const uint32_t before = inc - s;
      const bool mine = (long long)before < krem && krem <= (long long)inc;
      if (mine) {
        long long k = krem - before;
        int d = 255 - 8 * lane;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (k <= (long long)c[u]) {
            d = 255 - 8 * lane - u;
            break;
          }
          k -= c[u];
        }
        S.prefix = prefix | ((uint64_t)d << shift);
        S.krem = k;
      }
    }
    __syncthreads();
  }
  return S.prefix;
}

// Ordered selection over values get(j) / indices idx(j), j < m in index order:
// every value > T, then the first `need` values == T; sel receives them in that
// order (above first).  Processes 4 consecutive entries per thread per round.
template <class Get, class Idx>
__device__ void select_ordered(const Get& get, const Idx& idx, int64_t m, double T, int64_t above_total,
                               int64_t need, uint32_t* __restrict__ sel, SelShared& S) {
  int64_t a_off = 0, t_off = 0;
  const int64_t per = 4LL * blockDim.x;
  for (int64_t base = 0; base < m; base += per) {
    const int64_t j0 = base + 4LL * threadIdx.x;
    double v[4];
    uint32_t na = 0, nt = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[u] = (j0 + u < m) ? get(j0 + u) : -1.0;
      na += v[u] > T;
      nt += v[u] == T;
    }
    uint32_t atot, ttot;
    const uint32_t ea = block_exclusive_scan(na, S.scan_tmp, &atot);
    const uint32_t et = block_exclusive_scan(nt, S.scan_tmp, &ttot);
    int64_t pa = a_off + ea, pt = t_off + et;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (v[u] > T) {
        sel[pa++] = idx(j0 + u);
      } else if (v[u] == T) {
        if (pt < need) sel[above_total + pt] = idx(j0 + u);
        ++pt;
      }
    }
    a_off += atot;
    t_off += ttot;
    if (t_off >= need && a_off >= above_total) break;
  }
}

__global__ void __launch_bounds__(kT2, 3)
k_rs_select(const uint8_t* __restrict__ in, int64_t in_fs, ResizeGeo G, const double* __restrict__ dark,
            const uint32_t* __restrict__ hist, int64_t K, double alpha, uint32_t* __restrict__ sel_all,
            double* __restrict__ airlight) {
  extern __shared__ double dsm[];
  double* cval = dsm;                                           // [kCap]
  uint32_t* cidx = reinterpret_cast<uint32_t*>(dsm + kCap);     // [kCap]
  __shared__ SelShared S;
  __shared__ double s_f[256];
  __shared__ int s_B;
  __shared__ long long s_ncand;
  const int f = blockIdx.x;
  const int64_t npx = (int64_t)G.H * G.W;
  const double* fd = dark + (int64_t)f * npx;
  uint32_t* sel = sel_all + (int64_t)f * K;
  for (int v = threadIdx.x; v < 256; v += kT2) s_f[v] = u8f(v);

  if (K >= npx) {  // estimation.py:74-75: every pixel, in index order
    for (int64_t i = threadIdx.x; i < npx; i += kT2) sel[i] = (uint32_t)i;
  } else {
    // bucket B holding the K-th largest value (warp 0, descending suffix counts)
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      constexpr int kPer = (kResizeBuckets + 31) / 32;  // 129 buckets per lane, lane 0 owns the top
      const uint32_t* fh = hist + (int64_t)f * kResizeBuckets;
      const int hi = kResizeBuckets - 1 - lane * kPer, lo = max(hi - kPer + 1, 0);
      uint32_t s = 0;
      for (int b = hi; b >= lo; --b) s += fh[b];
      uint32_t inc = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const uint32_t before = inc - s;
      if ((int64_t)before < K && K <= (int64_t)inc) {
        uint32_t acc = before;
        for (int b = hi; b >= lo; --b) {
          acc += fh[b];
          if ((int64_t)acc >= K) {
            s_B = b;
            s_ncand = acc;
            break;
          }
        }
      }
    }
    __syncthreads();
    const int B = s_B;
    const int64_t ncand = s_ncand;
    uint64_t tkey;
    int64_t above_total = 0;
    if (ncand <= kCap) {
      // ordered compaction of the candidates (bucket >= B) into shared memory
      int64_t off = 0;
      for (int64_t base = 0; base < npx; base += 4LL * kT2) {
        const int64_t i0 = base + 4LL * threadIdx.x;
        double v[4];
        uint32_t c = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] = (i0 + u < npx) ? fd[i0 + u] : -1.0;
          c += (i0 + u < npx) && bucket_of(v[u]) >= B;
        }
        uint32_t tot;
        int64_t p = off + block_exclusive_scan(c, S.scan_tmp, &tot);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if ((i0 + u < npx) && bucket_of(v[u]) >= B) {
            cval[p] = v[u];
            cidx[p] = (uint32_t)(i0 + u);
            ++p;
          }
        off += tot;
        if (off >= ncand) break;
      }
      __syncthreads();
      auto get = [&](int64_t j) { return cval[j]; };
      auto idx = [&](int64_t j) { return cidx[j]; };
      tkey = radix_kth(get, ncand, K, S);
      const double T = __longlong_as_double((long long)(tkey & 0x7fffffffffffffffull));
      uint32_t na = 0;
      for (int64_t j = threadIdx.x; j < ncand; j += kT2) na += cval[j] > T;
      uint32_t tot;
      block_exclusive_scan(na, S.scan_tmp, &tot);
      above_total = tot;
      select_ordered(get, idx, ncand, T, above_total, K - above_total, sel, S);
    } else {
      // too many candidates for shared memory: the same steps over the whole frame
      auto get = [&](int64_t j) { return fd[j]; };
      auto idx = [&](int64_t j) { return (uint32_t)j; };
      tkey = radix_kth(get, npx, K, S);
      const double T = __longlong_as_double((long long)(tkey & 0x7fffffffffffffffull));
      uint32_t na = 0;
      for (int64_t j = threadIdx.x; j < npx; j += kT2) na += fd[j] > T;
      uint32_t tot;
      block_exclusive_scan(na, S.scan_tmp, &tot);
      above_total = tot;
      select_ordered(get, idx, npx, T, above_total, K - above_total, sel, S);
    }
  }
  __syncthreads();

  // airlight: sequential fp64 sum per channel in selection order (estimation.py:83-84)
  constexpr int kChunk = 1024;
  double* rgbs = dsm;  // [kChunk][3], reuses the candidate buffer
  const uint8_t* frame = in + (int64_t)f * in_fs;
  double acc = 0.0;
  for (int64_t base = 0; base < K; base += kChunk) {
    const int cnt = (int)min((int64_t)kChunk, K - base);
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += kT2) {
      const uint32_t p = sel[base + e];
      const int y = (int)(p / (uint32_t)G.W), x = (int)(p - (uint32_t)y * (uint32_t)G.W);
      double rgb[3];
      resized_rgb(frame, G, y, x, s_f, rgb);
      rgbs[3 * e] = rgb[0];
      rgbs[3 * e + 1] = rgb[1];
      rgbs[3 * e + 2] = rgb[2];
    }
    __syncthreads();
    if (threadIdx.x < 3)
      for (int e = 0; e < cnt; ++e) acc = __dadd_rn(acc, rgbs[3 * e + threadIdx.x]);
  }
  if (threadIdx.x < 3) {
    const double mean = __ddiv_rn(acc, (double)K);
    airlight[3 * f + threadIdx.x] = dmax(__dmul_rn(alpha, mean), 1e-6);
  }
}

// ------------------------------------------------------------------- R3 ----
// MODE 0: bytes from the global thresholds.  MODE 1: per-CTA channel sums of the
// gamma values (gray-world).  MODE 2: bytes from per-frame, per-channel thresholds.
template <int MODE>
__global__ void __launch_bounds__(kT3)
k_rs_recover(const uint8_t* __restrict__ in, int64_t in_fs, ResizeGeo G, const double* __restrict__ airlight,
             double omega, double t_min, const double* __restrict__ thr, const float* __restrict__ gains,
             double inv_gamma, int gamma_is_one, uint8_t* __restrict__ out, int64_t out_fs,
             double* __restrict__ part, int nframes) {
  __shared__ double s_f[256];
  __shared__ double s_thr[MODE == 2 ? 3 : 1][256];
  __shared__ double red[3][kT3 / 32];
  __shared__ TapS s_tx[kColTab];
  __shared__ PowTables PT;  // balance sums (MODE 1)
  __shared__ ByteBuckets BK;  // fp32 fast path of the bytes (MODE 0)
  // MODE 0 (nframes > 0): persistent CTAs over the batch's flat (frame, row) space — the
  // tables do not depend on the frame, so a CTA walks from frame to frame and every SM
  // keeps the same number of resident CTAs to the end (a (row block, frame) grid left a
  // thin last wave).  MODE 1 / 2: blockIdx.y is the frame, blockIdx.x its row block.
  int f = (MODE == 0) ? 0 : (int)blockIdx.y;
  s_f[threadIdx.x] = u8f(threadIdx.x);
  if (MODE == 1) pow_tables_init(PT);
  if (MODE == 0) s_thr[0][threadIdx.x] = thr[threadIdx.x];
  if (MODE == 2)
    for (int c = 0; c < 3; ++c) s_thr[c][threadIdx.x] = thr[((int64_t)f * 3 + c) * 256 + threadIdx.x];
  __syncthreads();
  if (MODE == 0) {
    byte_buckets_build(BK, s_thr[0]);
    __syncthreads();
  }
  const float ig = (float)inv_gamma;
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  // flat rows [q0, q1) (MODE 0: of the batch; else of the frame); column taps tabulated once per CTA
  const int64_t rows = (MODE == 0) ? (int64_t)nframes * G.H : (int64_t)G.H;
  const int64_t q0 = rows * blockIdx.x / gridDim.x, q1 = rows * (blockIdx.x + 1) / gridDim.x;
  const bool tab = G.W <= kColTab;
  for (int x = threadIdx.x; tab && x < G.W; x += kT3) s_tx[x] = compact(tap(x, G.sx, G.w));
  __syncthreads();
  for (int64_t q = q0; q < q1;) {
  if (MODE == 0) f = (int)(q / G.H);
  const int r0 = (int)(q - (int64_t)(MODE == 0 ? f : 0) * G.H);
  const int r1 = (int)min((int64_t)G.H, r0 + (q1 - q));
  q += r1 - r0;
  const double A0 = airlight[3 * f], A1 = airlight[3 * f + 1], A2 = airlight[3 * f + 2];
  const double amax = dmax(dmax(A0, A1), A2);
  const double ramax = __drcp_rn(amax);  // cmin / amax as the exact div_rb
  const float af0 = (float)A0, af1 = (float)A1, af2 = (float)A2;
  float g0 = 1.0f, g1 = 1.0f, g2 = 1.0f;
  if (MODE == 2) {
    g0 = gains[3 * f];
    g1 = gains[3 * f + 1];
    g2 = gains[3 * f + 2];
  }
  const uint8_t* frame = in + (int64_t)f * in_fs;
  uint8_t* fo = out + (int64_t)f * out_fs;
  for (int y = r0; y < r1; ++y)
  for (int x = threadIdx.x; x < G.W; x += kT3) {
    const int64_t p = (int64_t)y * G.W + x;
    double rgb[3];
    resized_rgb_t(frame, G.w, tap(y, G.sy, G.h), tab ? expand(s_tx[x], G.w) : tap(x, G.sx, G.w), s_f, rgb);
    const double cmin = dmin(dmin(rgb[0], rgb[1]), rgb[2]);
    if (MODE == 0) {
      // fp32 fast path (byte_bucket): t~ to ~1e-16 is plenty for it; the exact t,
      // recovery and thresholds only for a sample near a byte boundary
      const double tq = dmin(dmax(__fma_rn(-omega, __dmul_rn(cmin, ramax), 1.0), t_min), 1.0);
      const float rtf = rcp_approx(__double2float_rn(tq));
      bool ok = true;
      uint32_t k0 = byte_bucket(BK, __fmaf_rn(__double2float_rn(__dsub_rn(rgb[0], A0)), rtf, af0), ok);
      uint32_t k1 = byte_bucket(BK, __fmaf_rn(__double2float_rn(__dsub_rn(rgb[1], A1)), rtf, af1), ok);
      uint32_t k2 = byte_bucket(BK, __fmaf_rn(__double2float_rn(__dsub_rn(rgb[2], A2)), rtf, af2), ok);
      if (!ok) {
        const double t = dmin(dmax(__dsub_rn(1.0, __dmul_rn(omega, div_rb(cmin, amax, ramax))), t_min), 1.0);
        const double rt = __drcp_rn(t);
        k0 = quantize_thr_from(recover_raw(rgb[0], A0, t, rt), s_thr[0], (int)k0);
        k1 = quantize_thr_from(recover_raw(rgb[1], A1, t, rt), s_thr[0], (int)k1);
        k2 = quantize_thr_from(recover_raw(rgb[2], A2, t, rt), s_thr[0], (int)k2);
      }
      uint8_t* o = fo + 3 * p;
      o[0] = (uint8_t)k0;
      o[1] = (uint8_t)k1;
      o[2] = (uint8_t)k2;
      continue;
    }
    const double t = dmin(dmax(__dsub_rn(1.0, __dmul_rn(omega, div_rb(cmin, amax, ramax))), t_min), 1.0);
    const double rt = __drcp_rn(t);
    const double x0 = recover_raw(rgb[0], A0, t, rt), x1 = recover_raw(rgb[1], A1, t, rt),
                 x2 = recover_raw(rgb[2], A2, t, rt);
    if (MODE == 1) {
      if (gamma_is_one) {
        acc0 = __dadd_rn(acc0, dmin(dmax(x0, 0.0), 1.0));
        acc1 = __dadd_rn(acc1, dmin(dmax(x1, 0.0), 1.0));
        acc2 = __dadd_rn(acc2, dmin(dmax(x2, 0.0), 1.0));
      } else {
        acc0 = __dadd_rn(acc0, pow_tab(x0, inv_gamma, PT));
        acc1 = __dadd_rn(acc1, pow_tab(x1, inv_gamma, PT));
        acc2 = __dadd_rn(acc2, pow_tab(x2, inv_gamma, PT));
      }
    } else {
      const double* t0 = s_thr[0];
      const double* t1 = s_thr[MODE == 2 ? 1 : 0];
      const double* t2 = s_thr[MODE == 2 ? 2 : 0];
      uint8_t* o = fo + 3 * p;
      o[0] = (uint8_t)quantize_thr_from(x0, t0, guess_byte(x0, ig, g0));
      o[1] = (uint8_t)quantize_thr_from(x1, t1, guess_byte(x1, ig, g1));
      o[2] = (uint8_t)quantize_thr_from(x2, t2, guess_byte(x2, ig, g2));
    }
  }
  }  // flat row ranges
  if (MODE == 1) {
    double v3[3] = {acc0, acc1, acc2};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < 3; ++c) v3[c] = __dadd_rn(v3[c], __shfl_xor_sync(0xffffffffu, v3[c], o));
    if ((threadIdx.x & 31) == 0)
      for (int c = 0; c < 3; ++c) red[c][threadIdx.x >> 5] = v3[c];
    __syncthreads();
    if (threadIdx.x < 3) {
      double s = 0.0;
      for (int w = 0; w < kT3 / 32; ++w) s = __dadd_rn(s, red[threadIdx.x][w]);
      part[((int64_t)f * gridDim.x + blockIdx.x) * 3 + threadIdx.x] = s;
    }
  }
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace

cudaError_t resize_dark(const uint8_t* in, int64_t in_fs, int n, const ResizeGeo& g, int r, double* dark,
                        uint32_t* hist, cudaStream_t st) {
  if (r < 1 || r > kResizeMaxRadius) return cudaErrorInvalidValue;
  const size_t smem = (size_t)((kTH + 2 * r) * (kTW + 2 * r) + (kTH + 2 * r) * kTW) * sizeof(double);
  // row minima in place; odd pitch (k_rs_dark_t PWP)
  const size_t smem_t = (size_t)(kTH + 2 * r) * ((kTW + 2 * r) | 1) * sizeof(double);
  dim3 grid((g.W + kTW - 1) / kTW, (g.H + kTH - 1) / kTH, n);
  auto launch = [&](auto kern) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
    if (e != cudaSuccess) return e;
    kern<<<grid, kT1, smem_t, st>>>(in, in_fs, g, dark, hist);
    return cudaGetLastError();
  };
  switch (r) {
    case 1: return launch(k_rs_dark_t<1>);
    case 2: return launch(k_rs_dark_t<2>);
    case 3: return launch(k_rs_dark_t<3>);
    case 4: return launch(k_rs_dark_t<4>);
    case 5: return launch(k_rs_dark_t<5>);
    case 6: return launch(k_rs_dark_t<6>);
    case 7: return launch(k_rs_dark_t<7>);
    case 8: return launch(k_rs_dark_t<8>);
    case 10: return launch(k_rs_dark_t<10>);
    case 15: return launch(k_rs_dark_t<15>);
    default: break;
  }
  cudaError_t e = cudaFuncSetAttribute(k_rs_dark, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_rs_dark<<<grid, kT1, smem, st>>>(in, in_fs, g, r, dark, hist);
  return cudaGetLastError();
}

cudaError_t resize_select(const uint8_t* in, int64_t in_fs, int n, const ResizeGeo& g, const double* dark,
                          const uint32_t* hist, int64_t K, double alpha, uint32_t* sel, double* airlight,
                          cudaStream_t st) {
  const size_t smem = (size_t)kCap * (sizeof(double) + sizeof(uint32_t));
  cudaError_t e = cudaFuncSetAttribute(k_rs_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_rs_select<<<n, kT2, smem, st>>>(in, in_fs, g, dark, hist, K, alpha, sel, airlight);
  return cudaGetLastError();
}

size_t resize_balance_ws_bytes(int n) {
  return (size_t)n * (kResizeSumParts * 3 * 8 + 3 * 256 * 8 + 16);
}

cudaError_t resize_recover(const uint8_t* in, int64_t in_fs, int n, const ResizeGeo& g, const double* airlight,
                           double omega, double t_min, const double* thr, double gamma, bool balance,
                           void* bal_ws, uint8_t* out, int64_t out_fs, cudaStream_t st) {
  const int64_t npx = (int64_t)g.H * g.W;
  const double ig = 1.0 / gamma;
  const int g1 = gamma == 1.0 ? 1 : 0;
  if (!balance) {
    // persistent: every SM's full complement of CTAs over the batch's flat rows (at least ~2 rows each)
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rs_recover<0>, kT3, 0);
    const int64_t rows = (int64_t)n * g.H;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(occ, 1) * sm_count(), (rows + 1) / 2));
    k_rs_recover<0><<<grid, kT3, 0, st>>>(in, in_fs, g, airlight, omega, t_min, thr, nullptr, ig, g1, out, out_fs,
                                          nullptr, n);
    return cudaGetLastError();
  }
  double* part = static_cast<double*>(bal_ws);
  double* bthr = part + (size_t)n * kResizeSumParts * 3;
  float* gains = reinterpret_cast<float*>(bthr + (size_t)n * 3 * 256);
  k_rs_recover<1><<<dim3(kResizeSumParts, n), kT3, 0, st>>>(in, in_fs, g, airlight, omega, t_min, nullptr, nullptr,
                                                            ig, g1, out, out_fs, part, n);
  cudaError_t e = balance_thresholds(part, kResizeSumParts, n, npx, gamma, bthr, gains, st);
  if (e != cudaSuccess) return e;
  k_rs_recover<2><<<dim3(kResizeSumParts, n), kT3, 0, st>>>(in, in_fs, g, airlight, omega, t_min, bthr, gains, ig,
                                                            g1, out, out_fs, nullptr, n);
  return cudaGetLastError();
}

}  // namespace dhz
