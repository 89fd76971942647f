// float64 device path: the reference's public stage functions on float64 arrays
// and the float pipeline used when frames are resized (reference default
// resize_to=(640, 480)) or refined by the guided filter (image mode).
//
// Every elementwise kernel keeps the reference's numpy operation order with one
// rounding per numpy op (__dadd_rn/__dmul_rn/__ddiv_rn: no FMA contraction), so
// the results are bit-identical to numpy wherever numpy itself is (everything
// but power(), whose device pow is within ~1 ulp, and the sum orders of means
// and box filters, which are deterministic here but not numpy's).
//   u8_to_float / float_to_u8 / to_grayscale / resize_bilinear   imageops.py:18-78
//   channel_min / estimate_airlight / transmission / box / guided  estimation.py:35-172
//   min_filter                                                   morphology.py:63-73
//   recover_radiance / gamma_correct / gray_world_balance        recover.py:28-69
#include <algorithm>
#include <cstdint>

#include "../../include/dehaze_b200.h"
#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

constexpr int kT = 256;

inline int grid_for(int64_t n, int per_thread = 1) {
  int64_t b = (n + (int64_t)kT * per_thread - 1) / ((int64_t)kT * per_thread);
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

#define GRID_STRIDE(i, n) for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); \
                               i += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ double clip01(double x) { return fmin(fmax(x, 0.0), 1.0); }

// ---------------------------------------------------------------- stats ----
// out[0] = 1 if every element is finite, out[1] = min, out[2] = max
__global__ void k_stats_partial(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double smin[kT], smax[kT];
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  double lo = INFINITY, hi = -INFINITY;
  bool bad = false;
  GRID_STRIDE(i, n) {
    const double v = x[i];
    if (!isfinite(v)) bad = true;
    lo = fmin(lo, v);
    hi = fmax(hi, v);
  }
  if (bad) sbad = 1;
  smin[threadIdx.x] = lo;
  smax[threadIdx.x] = hi;
  __syncthreads();
  for (int s = kT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + s]);
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = sbad ? 0.0 : 1.0;
    part[3 * blockIdx.x + 1] = smin[0];
    part[3 * blockIdx.x + 2] = smax[0];
  }
}
__global__ void k_stats_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double ok = 1.0, lo = INFINITY, hi = -INFINITY;
  for (int b = 0; b < nb; ++b) {
    ok = fmin(ok, part[3 * b]);
    lo = fmin(lo, part[3 * b + 1]);
    hi = fmax(hi, part[3 * b + 2]);
  }
  out[0] = ok;
  out[1] = lo;
  out[2] = hi;
}

// ------------------------------------------------------------ conversions ----
__global__ void k_u8_to_f64(const uint8_t* __restrict__ in, int64_t n, double* __restrict__ out) {
  GRID_STRIDE(i, n) out[i] = __ddiv_rn((double)in[i], 255.0);
}
__global__ void k_f64_to_u8(const double* __restrict__ in, int64_t n, uint8_t* __restrict__ out) {
  GRID_STRIDE(i, n) out[i] = (uint8_t)quantize_unit(in[i]);
}
__global__ void k_gray(const double* __restrict__ img, int64_t npx, double* __restrict__ out) {
  GRID_STRIDE(p, npx) {
    const double r = img[3 * p], g = img[3 * p + 1], b = img[3 * p + 2];
    const double v = __dadd_rn(__dadd_rn(__dmul_rn(0.299, r), __dmul_rn(0.587, g)), __dmul_rn(0.114, b));
    out[p] = clip01(v);
  }
}
__global__ void k_channel_min(const double* __restrict__ img, int64_t npx, double* __restrict__ out) {
  GRID_STRIDE(p, npx) out[p] = fmin(fmin(img[3 * p], img[3 * p + 1]), img[3 * p + 2]);
}

// --------------------------------------------------------------- resize ----
// pixel-centre bilinear (imageops.py:64-78): rows blend first, then columns.
template <typename Src>
__global__ void k_resize(const Src* __restrict__ in, int h, int w, int height, int width, double sy_scale,
                         double sx_scale, double* __restrict__ out) {
  const int64_t n = (int64_t)height * width * 3;
  GRID_STRIDE(i, n) {
    const int c = (int)(i % 3);
    const int64_t px = i / 3;
    const int y = (int)(px / width), x = (int)(px - (int64_t)y * width);
    double sy = __dsub_rn(__dmul_rn(__dadd_rn((double)y, 0.5), sy_scale), 0.5);
    double sx = __dsub_rn(__dmul_rn(__dadd_rn((double)x, 0.5), sx_scale), 0.5);
    sy = fmin(fmax(sy, 0.0), (double)h - 1.0);
    sx = fmin(fmax(sx, 0.0), (double)w - 1.0);
    const int y0 = (int)floor(sy), x0 = (int)floor(sx);
    const int y1 = min(y0 + 1, h - 1), x1 = min(x0 + 1, w - 1);
    const double fy = __dsub_rn(sy, (double)y0), fx = __dsub_rn(sx, (double)x0);
    const double gy = __dsub_rn(1.0, fy), gx = __dsub_rn(1.0, fx);
    auto val = [&](int yy, int xx) -> double {
      const double v = (double)in[((int64_t)yy * w + xx) * 3 + c];
      return sizeof(Src) == 1 ? __ddiv_rn(v, 255.0) : v;
    };
    const double r0 = __dadd_rn(__dmul_rn(val(y0, x0), gy), __dmul_rn(val(y1, x0), fy));
    const double r1 = __dadd_rn(__dmul_rn(val(y0, x1), gy), __dmul_rn(val(y1, x1), fy));
    out[i] = clip01(__dadd_rn(__dmul_rn(r0, gx), __dmul_rn(r1, fx)));
  }
}

// Direct-window oracles of the reference's correctness references, independent of
// the separable kernels above: every output scans its own (2r+1)^2 window of the
// edge-padded map.  morphology.py:76-92 (min; exact in any order) and
// estimation.py:128-141 (window mean: a row-major sequential sum / k^2 here, numpy
// sums pairwise; the reference tests compare with a 1e-6 tolerance).
__global__ void k_min_naive(const double* __restrict__ m, int H, int W, int r, double* __restrict__ out) {
  const int64_t n = (int64_t)H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / W), x = (int)(i - (int64_t)y * W);
    double v = m[i];
    for (int dy = -r; dy <= r; ++dy) {
      const double* row = m + (int64_t)min(max(y + dy, 0), H - 1) * W;
      for (int dx = -r; dx <= r; ++dx) v = fmin(v, row[min(max(x + dx, 0), W - 1)]);
    }
    out[i] = v;
  }
}

__global__ void k_box_naive(const double* __restrict__ m, int H, int W, int r, double kk, double* __restrict__ out) {
  const int64_t n = (int64_t)H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / W), x = (int)(i - (int64_t)y * W);
    double s = 0.0;
    for (int dy = -r; dy <= r; ++dy) {
      const double* row = m + (int64_t)min(max(y + dy, 0), H - 1) * W;
      for (int dx = -r; dx <= r; ++dx) s = __dadd_rn(s, row[min(max(x + dx, 0), W - 1)]);
    }
    out[i] = __ddiv_rn(s, kk);
  }
}

// ----------------------------------------------------------- min filter ----
__global__ void k_min_rows(const double* __restrict__ m, int H, int W, int r, double* __restrict__ out) {
  const int64_t n = (int64_t)H * W;
  GRID_STRIDE(i, n) {
    const int y = (int)(i / W), x = (int)(i - (int64_t)y * W);
    const double* row = m + (int64_t)y * W;
    double v = row[x];
    for (int k = max(0, x - r); k <= min(W - 1, x + r); ++k) v = fmin(v, row[k]);
    out[i] = v;
  }
}
__global__ void k_min_cols(const double* __restrict__ m, int H, int W, int r, double* __restrict__ out) {
  const int64_t n = (int64_t)H * W;
  GRID_STRIDE(i, n) {
    const int y = (int)(i / W), x = (int)(i - (int64_t)y * W);
    double v = m[i];
    for (int k = max(0, y - r); k <= min(H - 1, y + r); ++k) v = fmin(v, m[(int64_t)k * W + x]);
    out[i] = v;
  }
}

// ----------------------------------------------------------- box filter ----
// Window sums with replicate borders, runs of kRunLen outputs per thread: the
// first sum of a run is direct (2r+1 adds), the rest slide (add new, drop old).
constexpr int kRunLen = 32;
__global__ void k_box_rows(const double* __restrict__ m, int H, int W, int r, double* __restrict__ out) {
  const int runs = (W + kRunLen - 1) / kRunLen;
  const int64_t n = (int64_t)H * runs;
  GRID_STRIDE(i, n) {
    const int y = (int)(i / runs), x0 = (int)(i - (int64_t)y * runs) * kRunLen;
    const double* row = m + (int64_t)y * W;
    double s = 0.0;
    for (int d = -r; d <= r; ++d) s = __dadd_rn(s, row[min(W - 1, max(0, x0 + d))]);
    out[(int64_t)y * W + x0] = s;
    for (int x = x0 + 1; x < min(W, x0 + kRunLen); ++x) {
      s = __dadd_rn(s, row[min(W - 1, x + r)]);
      s = __dsub_rn(s, row[max(0, x - r - 1)]);
      out[(int64_t)y * W + x] = s;
    }
  }
}
__global__ void k_box_cols(const double* __restrict__ m, int H, int W, int r, double inv_div_unused, double div,
                           double* __restrict__ out) {
  const int runs = (H + kRunLen - 1) / kRunLen;
  const int64_t n = (int64_t)W * runs;
  GRID_STRIDE(i, n) {
    const int run = (int)(i / W), x = (int)(i - (int64_t)run * W);
    const int y0 = run * kRunLen;
    double s = 0.0;
    for (int d = -r; d <= r; ++d) s = __dadd_rn(s, m[(int64_t)min(H - 1, max(0, y0 + d)) * W + x]);
    out[(int64_t)y0 * W + x] = __ddiv_rn(s, div);
    for (int y = y0 + 1; y < min(H, y0 + kRunLen); ++y) {
      s = __dadd_rn(s, m[(int64_t)min(H - 1, y + r) * W + x]);
      s = __dsub_rn(s, m[(int64_t)max(0, y - r - 1) * W + x]);
      out[(int64_t)y * W + x] = __ddiv_rn(s, div);
    }
  }
}

// ------------------------------------------------------- guided filter ----
__global__ void k_gf_products(const double* __restrict__ p, const double* __restrict__ g, int64_t n,
                              double* __restrict__ gp, double* __restrict__ gg) {
  GRID_STRIDE(i, n) {
    gp[i] = __dmul_rn(g[i], p[i]);
    gg[i] = __dmul_rn(g[i], g[i]);
  }
}
__global__ void k_gf_ab(const double* __restrict__ mi, const double* __restrict__ mp, const double* __restrict__ cip,
                        const double* __restrict__ cii, int64_t n, double eps, double* __restrict__ a,
                        double* __restrict__ b) {
  GRID_STRIDE(i, n) {
    const double var = __dsub_rn(cii[i], __dmul_rn(mi[i], mi[i]));
    const double cov = __dsub_rn(cip[i], __dmul_rn(mi[i], mp[i]));
    const double av = __ddiv_rn(cov, __dadd_rn(var, eps));
    a[i] = av;
    b[i] = __dsub_rn(mp[i], __dmul_rn(av, mi[i]));
  }
}
__global__ void k_gf_out(const double* __restrict__ ma, const double* __restrict__ mb, const double* __restrict__ g,
                         int64_t n, double floor_t, double* __restrict__ q) {
  GRID_STRIDE(i, n) {
    const double v = clip01(__dadd_rn(__dmul_rn(ma[i], g[i]), mb[i]));
    q[i] = floor_t > 0.0 ? fmax(v, floor_t) : v;  // pipeline.py:203 re-floor when requested
  }
}

// ------------------------------------------------ transmission / recover ----
__global__ void k_transmission(const double* __restrict__ cmin, int64_t n, const double* __restrict__ A,
                               double omega, double t_min, double* __restrict__ t) {
  const double amax = fmax(fmax(A[0], A[1]), A[2]);
  GRID_STRIDE(i, n) {
    const double v = __dsub_rn(1.0, __dmul_rn(omega, __ddiv_rn(cmin[i], amax)));
    t[i] = fmin(fmax(v, t_min), 1.0);
  }
}
__device__ __forceinline__ double recover1(double I, double A, double t) {
  return clip01(__dadd_rn(__ddiv_rn(__dsub_rn(I, A), t), A));
}
__global__ void k_recover(const double* __restrict__ img, const double* __restrict__ A, const double* __restrict__ t,
                          int64_t npx, double* __restrict__ out) {
  const double A0 = A[0], A1 = A[1], A2 = A[2];
  GRID_STRIDE(p, npx) {
    const double tt = t[p];
    out[3 * p] = recover1(img[3 * p], A0, tt);
    out[3 * p + 1] = recover1(img[3 * p + 1], A1, tt);
    out[3 * p + 2] = recover1(img[3 * p + 2], A2, tt);
  }
}
// recover -> gamma -> u8 in one pass, exact through the host threshold table
__global__ void k_recover_quant(const double* __restrict__ img, const double* __restrict__ A,
                                const double* __restrict__ t, int64_t npx, const double* __restrict__ thr,
                                uint8_t* __restrict__ out) {
  __shared__ double s_thr[256];
  for (int v = threadIdx.x; v < 256; v += blockDim.x) s_thr[v] = thr[v];
  __syncthreads();
  const double A0 = A[0], A1 = A[1], A2 = A[2];
  GRID_STRIDE(p, npx) {
    const double tt = t[p];
    out[3 * p] = (uint8_t)quantize_thr(recover1(img[3 * p], A0, tt), s_thr);
    out[3 * p + 1] = (uint8_t)quantize_thr(recover1(img[3 * p + 1], A1, tt), s_thr);
    out[3 * p + 2] = (uint8_t)quantize_thr(recover1(img[3 * p + 2], A2, tt), s_thr);
  }
}
__global__ void k_gamma(const double* __restrict__ in, int64_t n, double e, double* __restrict__ out) {
  GRID_STRIDE(i, n) out[i] = clip01(pow(in[i], e));
}

// -------------------------------------------------------- gray world ----
__global__ void k_channel_sums(const double* __restrict__ img, int64_t npx, double* __restrict__ part) {
  __shared__ double s[3][kT];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  // contiguous chunk per block, strided within: a fixed, launch-independent order
  const int64_t per = (npx + gridDim.x - 1) / gridDim.x;
  const int64_t p0 = (int64_t)blockIdx.x * per, p1 = min(npx, p0 + per);
  for (int64_t p = p0 + threadIdx.x; p < p1; p += kT) {
    a0 = __dadd_rn(a0, img[3 * p]);
    a1 = __dadd_rn(a1, img[3 * p + 1]);
    a2 = __dadd_rn(a2, img[3 * p + 2]);
  }
  s[0][threadIdx.x] = a0;
  s[1][threadIdx.x] = a1;
  s[2][threadIdx.x] = a2;
  __syncthreads();
  for (int k = kT / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k)
      for (int c = 0; c < 3; ++c) s[c][threadIdx.x] = __dadd_rn(s[c][threadIdx.x], s[c][threadIdx.x + k]);
    __syncthreads();
  }
  if (threadIdx.x < 3) part[3 * blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}
// gains[0..2]; gains[3] = 1 when the frame is left unchanged (a channel mean < 1e-6)
__global__ void k_gains(const double* __restrict__ part, int nb, int64_t npx, double* __restrict__ gains) {
  if (threadIdx.x != 0) return;
  double m[3];
  for (int c = 0; c < 3; ++c) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s = __dadd_rn(s, part[3 * b + c]);
    m[c] = __ddiv_rn(s, (double)npx);
  }
  const bool degenerate = fmin(fmin(m[0], m[1]), m[2]) < 1e-6;
  const double mm = __ddiv_rn(__dadd_rn(__dadd_rn(m[0], m[1]), m[2]), 3.0);
  for (int c = 0; c < 3; ++c) gains[c] = degenerate ? 1.0 : fmin(fmax(__ddiv_rn(mm, m[c]), 0.5), 2.0);
  gains[3] = degenerate ? 1.0 : 0.0;
}
__global__ void k_apply_gains(const double* __restrict__ img, int64_t npx, const double* __restrict__ gains,
                              double* __restrict__ out) {
  const bool copy = gains[3] != 0.0;
  const double g0 = gains[0], g1 = gains[1], g2 = gains[2];
  GRID_STRIDE(p, npx) {
    if (copy) {
      out[3 * p] = img[3 * p];
      out[3 * p + 1] = img[3 * p + 1];
      out[3 * p + 2] = img[3 * p + 2];
    } else {
      out[3 * p] = clip01(__dmul_rn(img[3 * p], g0));
      out[3 * p + 1] = clip01(__dmul_rn(img[3 * p + 1], g1));
      out[3 * p + 2] = clip01(__dmul_rn(img[3 * p + 2], g2));
    }
  }
}

// ------------------------------------------------------ airlight (f64) ----
// Order-preserving key of a double (-0.0 folded onto +0.0, as numpy compares them equal).
__device__ __forceinline__ uint64_t dkey(double d) {
  uint64_t b = (uint64_t)__double_as_longlong(d == 0.0 ? 0.0 : d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

constexpr int kSelT = 1024;

// One CTA: radix-select the K-th largest key (8 passes of 8 bits), then the
// ordered compaction (above in index order, then the first K-above ties) and the
// three sequential fp64 channel sums (estimation.py:71-84).
__global__ void __launch_bounds__(kSelT)
k_airlight_f64(const double* __restrict__ img, const double* __restrict__ dark, int64_t n, int64_t K,
               double alpha, double* __restrict__ A, uint32_t* __restrict__ sel) {
  __shared__ uint32_t hist[kSelT / 32][256];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_krem;
  __shared__ uint32_t tmp[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (K >= n) {  // arange(n)
    for (int64_t i = threadIdx.x; i < n; i += kSelT) sel[i] = (uint32_t)i;
  } else {
    if (threadIdx.x == 0) {
      s_prefix = 0;
      s_krem = K;
    }
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
      for (int k = threadIdx.x; k < (kSelT / 32) * 256; k += kSelT) (&hist[0][0])[k] = 0;
      __syncthreads();
      const uint64_t prefix = s_prefix;
      const uint64_t pmask = pass == 0 ? 0ull : (~0ull << (64 - 8 * pass));
      for (int64_t i = threadIdx.x; i < n; i += kSelT) {
        const uint64_t key = dkey(dark[i]);
        if ((key & pmask) == prefix) atomicAdd(&hist[wid][(key >> shift) & 0xFFu], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 256) {
        uint32_t s = 0;
        for (int w = 0; w < kSelT / 32; ++w) s += hist[w][threadIdx.x];
        hist[0][threadIdx.x] = s;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int64_t krem = s_krem;
        int d = 255;
        for (; d > 0; --d) {
          if ((int64_t)hist[0][d] >= krem) break;
          krem -= hist[0][d];
        }
        s_prefix = prefix | ((uint64_t)d << shift);
        s_krem = krem;
      }
      __syncthreads();
    }
    const uint64_t T = s_prefix;
    // above = #(key > T); ties needed = K - above
    uint32_t na = 0;
    for (int64_t i = threadIdx.x; i < n; i += kSelT) na += dkey(dark[i]) > T;
    uint32_t above;
    block_exclusive_scan(na, tmp, &above);
    const uint32_t need = (uint32_t)K - above;
    uint32_t abase = 0, tbase = 0;
    for (int64_t c0 = 0; c0 < n; c0 += kSelT) {
      const int64_t i = c0 + threadIdx.x;
      const uint64_t key = i < n ? dkey(dark[i]) : 0ull;
      const uint32_t fa = i < n && key > T, ft = i < n && key == T;
      uint32_t ta, tt;
      const uint32_t pa = block_exclusive_scan(fa, tmp, &ta);
      const uint32_t pt = block_exclusive_scan(ft, tmp, &tt);
      if (fa) sel[abase + pa] = (uint32_t)i;
      if (ft && tbase + pt < need) sel[above + tbase + pt] = (uint32_t)i;
      abase += ta;
      tbase += tt;
    }
    (void)lane;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int64_t k = 0; k < K; ++k) acc = __dadd_rn(acc, img[3 * (int64_t)sel[k] + threadIdx.x]);
    A[threadIdx.x] = fmax(__dmul_rn(alpha, __ddiv_rn(acc, (double)K)), 1e-6);
  }
}

}  // namespace
}  // namespace dhz

// =============================================================== C ABI ====
namespace {
inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int ret(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DHZ_OK : dhz::abi_cuda_fail(e, what);
}
}  // namespace

using namespace dhz;

extern "C" {

int dhz_f64_stats(const double* x, int64_t n, double* out3, double* ws, void* stream) {
  const int nb = std::min(grid_for(n), 1024);
  k_stats_partial<<<nb, kT, 0, S(stream)>>>(x, n, ws);
  k_stats_final<<<1, 32, 0, S(stream)>>>(ws, nb, out3);
  return ret("f64_stats");
}
int dhz_u8_to_f64(const uint8_t* in, int64_t n, double* out, void* stream) {
  k_u8_to_f64<<<grid_for(n), kT, 0, S(stream)>>>(in, n, out);
  return ret("u8_to_f64");
}
int dhz_f64_to_u8(const double* in, int64_t n, uint8_t* out, void* stream) {
  k_f64_to_u8<<<grid_for(n), kT, 0, S(stream)>>>(in, n, out);
  return ret("f64_to_u8");
}
int dhz_to_grayscale_f64(const double* img, int64_t npx, double* out, void* stream) {
  k_gray<<<grid_for(npx), kT, 0, S(stream)>>>(img, npx, out);
  return ret("to_grayscale_f64");
}
int dhz_channel_min_f64(const double* img, int64_t npx, double* out, void* stream) {
  k_channel_min<<<grid_for(npx), kT, 0, S(stream)>>>(img, npx, out);
  return ret("channel_min_f64");
}
int dhz_resize_bilinear_f64(const double* in, int h, int w, int height, int width, double* out, void* stream) {
  const double sy = (double)h / (double)height, sx = (double)w / (double)width;
  k_resize<double><<<grid_for((int64_t)height * width * 3), kT, 0, S(stream)>>>(in, h, w, height, width, sy, sx, out);
  return ret("resize_bilinear_f64");
}
int dhz_resize_bilinear_u8(const uint8_t* in, int h, int w, int height, int width, double* out, void* stream) {
  const double sy = (double)h / (double)height, sx = (double)w / (double)width;
  k_resize<uint8_t><<<grid_for((int64_t)height * width * 3), kT, 0, S(stream)>>>(in, h, w, height, width, sy, sx,
                                                                                 out);
  return ret("resize_bilinear_u8");
}
int dhz_min_filter_naive_f64(const double* m, int H, int W, int r, double* out, void* stream) {
  k_min_naive<<<grid_for((int64_t)H * W), kT, 0, S(stream)>>>(m, H, W, r, out);
  return ret("min_filter_naive_f64");
}
int dhz_box_filter_naive_f64(const double* m, int H, int W, int r, double* out, void* stream) {
  const double k = 2.0 * r + 1.0;
  k_box_naive<<<grid_for((int64_t)H * W), kT, 0, S(stream)>>>(m, H, W, r, k * k, out);
  return ret("box_filter_naive_f64");
}
int dhz_min_filter_f64(const double* m, int H, int W, int r, double* out, double* tmp, void* stream) {
  const int64_t n = (int64_t)H * W;
  k_min_rows<<<grid_for(n), kT, 0, S(stream)>>>(m, H, W, r, tmp);
  k_min_cols<<<grid_for(n), kT, 0, S(stream)>>>(tmp, H, W, r, out);
  return ret("min_filter_f64");
}
int dhz_box_filter_f64(const double* m, int H, int W, int r, double* out, double* tmp, void* stream) {
  const double k = 2.0 * r + 1.0;
  k_box_rows<<<grid_for((int64_t)H * ((W + kRunLen - 1) / kRunLen)), kT, 0, S(stream)>>>(m, H, W, r, tmp);
  k_box_cols<<<grid_for((int64_t)W * ((H + kRunLen - 1) / kRunLen)), kT, 0, S(stream)>>>(tmp, H, W, r, 0.0,
                                                                                          k * k, out);
  return ret("box_filter_f64");
}
int dhz_guided_filter_f64(const double* p, const double* guide, int H, int W, int r, double eps, double floor_t,
                          double* out, double* ws, void* stream) {
  const int64_t n = (int64_t)H * W;
  double* gp = ws;
  double* gg = ws + n;
  double* mi = ws + 2 * n;
  double* mp = ws + 3 * n;
  double* cip = ws + 4 * n;
  double* cii = ws + 5 * n;
  double* tmp = ws + 6 * n;
  double* a = gp;   // reuse after the products are boxed
  double* b = gg;
  k_gf_products<<<grid_for(n), kT, 0, S(stream)>>>(p, guide, n, gp, gg);
  int rc;
  if ((rc = dhz_box_filter_f64(guide, H, W, r, mi, tmp, stream))) return rc;
  if ((rc = dhz_box_filter_f64(p, H, W, r, mp, tmp, stream))) return rc;
  if ((rc = dhz_box_filter_f64(gp, H, W, r, cip, tmp, stream))) return rc;
  if ((rc = dhz_box_filter_f64(gg, H, W, r, cii, tmp, stream))) return rc;
  k_gf_ab<<<grid_for(n), kT, 0, S(stream)>>>(mi, mp, cip, cii, n, eps, a, b);
  if ((rc = dhz_box_filter_f64(a, H, W, r, mi, tmp, stream))) return rc;
  if ((rc = dhz_box_filter_f64(b, H, W, r, mp, tmp, stream))) return rc;
  k_gf_out<<<grid_for(n), kT, 0, S(stream)>>>(mi, mp, guide, n, floor_t, out);
  return ret("guided_filter_f64");
}
int dhz_transmission_f64(const double* cmin, int64_t npx, const double* airlight, double omega, double t_min,
                         double* out, void* stream) {
  k_transmission<<<grid_for(npx), kT, 0, S(stream)>>>(cmin, npx, airlight, omega, t_min, out);
  return ret("transmission_f64");
}
int dhz_recover_f64(const double* img, const double* airlight, const double* t, int64_t npx, double* out,
                    void* stream) {
  k_recover<<<grid_for(npx), kT, 0, S(stream)>>>(img, airlight, t, npx, out);
  return ret("recover_f64");
}
int dhz_recover_quant_f64(const double* img, const double* airlight, const double* t, int64_t npx,
                          const double* thresholds, uint8_t* out, void* stream) {
  k_recover_quant<<<grid_for(npx), kT, 0, S(stream)>>>(img, airlight, t, npx, thresholds, out);
  return ret("recover_quant_f64");
}
int dhz_gamma_f64(const double* in, int64_t n, double gamma, double* out, void* stream) {
  k_gamma<<<grid_for(n), kT, 0, S(stream)>>>(in, n, 1.0 / gamma, out);
  return ret("gamma_f64");
}
int dhz_gray_world_f64(const double* img, int64_t npx, double* out, double* ws, void* stream) {
  const int nb = 256;
  k_channel_sums<<<nb, kT, 0, S(stream)>>>(img, npx, ws);
  k_gains<<<1, 32, 0, S(stream)>>>(ws, nb, npx, ws + 3 * nb);
  k_apply_gains<<<grid_for(npx), kT, 0, S(stream)>>>(img, npx, ws + 3 * nb, out);
  return ret("gray_world_f64");
}
int dhz_airlight_f64(const double* img, const double* dark, int64_t npx, int64_t K, double alpha, double* airlight,
                     uint32_t* sel, void* stream) {
  if (K < 1 || K > npx) return dhz::abi_fail(DHZ_E_INVALID, "K out of range");
  k_airlight_f64<<<1, kSelT, 0, S(stream)>>>(img, dark, npx, K, alpha, airlight, sel);
  return ret("airlight_f64");
}

}  // extern "C"
