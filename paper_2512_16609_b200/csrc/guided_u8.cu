// Image mode on u8 frames at native resolution: guided-filter refinement of the
// transmission map fused with recovery (reference estimation.py:144-172,
// pipeline.py:197-215, imageops.py:39-44).
//
// Inputs per frame: the u8 frame and its airlight A (from K2-K4, bit-exact).
//   p(x)   = t_coarse = clip(1 - omega * (m/255) / max(A), t_min, 1)   (256-entry table of m)
//   g(x)   = clip((0.299*R' + 0.587*G') + 0.114*B', 0, 1), R' = R/255      (exact fp64 ops)
//   mean_I, mean_p, corr_Ip, corr_II = box_r(g), box_r(p), box_r(g*p), box_r(g*g)
//   a = (corr_Ip - mean_I*mean_p) / ((corr_II - mean_I^2) + eps),  b = mean_p - a*mean_I
//   t~ = max(clip(box_r(a) * g + box_r(b), 0, 1), t_min)
//   out_c = float_to_u8(gamma(clip((I_c' - A_c) / t~ + A_c)))  [* gray-world gains]
//
// Box sums (replicate border == clamped indices, divisor (2r+1)^2 like the
// reference's SAT) run as column-strip sliding sums: a CTA owns 256 input
// columns (256-2r output columns) and a segment of rows; each thread keeps the
// vertical window sums of its column in fp64 registers (add the entering row,
// drop the leaving one), and every output row takes its horizontal windows from
// a shared-memory fp64 prefix sum over the 256 columns.  Pass 1 writes a, b
// (fp64, 16 B/px); pass 2 boxes them, forms t~ and recovers the output bytes
// directly (exact thresholds), or — with gray-world balance — writes t~ and
// per-CTA channel sums of the gamma values for the apply pass.
#include <algorithm>

#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

constexpr int kCols = 256;   // input columns per CTA (one per thread)

__device__ __forceinline__ double u8f(uint32_t v) { return __ddiv_rn((double)v, 255.0); }

// Correctly rounded a / b from rb = RN(1/b): q0 = RN(a*rb) lies within 1 ulp of
// a/b, the FMA residual a - b*q0 is exact, and one correction step rounds to
// RN(a/b) (Markstein's theorem; b here is a positive normal constant).
__device__ __forceinline__ double div_rb(double a, double b, double rb) {
  const double q = __dmul_rn(a, rb);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, rb, q);
}

// Per-CTA tables: exact u8 -> fp64 products used by the guide and the coarse t.
struct GuideTables {
  double wr[256], wg[256], wb[256];  // 0.299*(v/255), 0.587*(v/255), 0.114*(v/255), one rounding each
  double t[256];                     // clip(1 - omega*((v/255)/max(A)), t_min, 1)
};

__device__ __forceinline__ void load_tables(GuideTables& T, const double* airlight, int f, double omega,
                                            double t_min) {
  const double amax = fmax(fmax(airlight[3 * f], airlight[3 * f + 1]), airlight[3 * f + 2]);
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    const double x = u8f(v);
    T.wr[v] = __dmul_rn(0.299, x);
    T.wg[v] = __dmul_rn(0.587, x);
    T.wb[v] = __dmul_rn(0.114, x);
    T.t[v] = fmin(fmax(__dsub_rn(1.0, __dmul_rn(omega, __ddiv_rn(x, amax))), t_min), 1.0);
  }
}

__device__ __forceinline__ double guide_t(const GuideTables& T, uint32_t r, uint32_t g, uint32_t b) {
  return fmin(fmax(__dadd_rn(__dadd_rn(T.wr[r], T.wg[g]), T.wb[b]), 0.0), 1.0);
}

// Warp-inclusive scan of NQ values, then the cross-warp carry from `wt` (one
// barrier); returns the CTA-inclusive prefix in v[].
template <int NQ>
__device__ __forceinline__ void cta_prefix(double (&v)[NQ], double (*wt)[kCols / 32]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double y = __shfl_up_sync(0xffffffffu, v[q], o);
      if (lane >= o) v[q] = __dadd_rn(v[q], y);
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) wt[q][wid] = v[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double base = 0.0;
    for (int w = 0; w < wid; ++w) base = __dadd_rn(base, wt[q][w]);
    v[q] = __dadd_rn(base, v[q]);
  }
}

// ---------------------------------------------------------------- pass 1 ----
// a, b for every pixel of the strip x in [x0, x0 + 256 - 2r), rows [y0, y0 + seg).
__global__ void __launch_bounds__(kCols)
k_gf_pass1(const uint8_t* __restrict__ in, int64_t in_fs, int H, int W, int r, int seg, double eps,
           const double* __restrict__ airlight, double omega, double t_min, double* __restrict__ a_out,
           double* __restrict__ b_out) {
  __shared__ GuideTables T;
  __shared__ double pre[2][4][kCols + 1];
  __shared__ double wt[2][4][kCols / 32];
  const int f = blockIdx.z;
  const int sw = kCols - 2 * r;                  // output columns of this strip
  const int x0 = blockIdx.x * sw;                // first output column
  const int y0 = blockIdx.y * seg;
  const int y1 = min(H, y0 + seg);
  load_tables(T, airlight, f, omega, t_min);
  if (threadIdx.x < 8) pre[threadIdx.x >> 2][threadIdx.x & 3][0] = 0.0;
  __syncthreads();
  const int xc = min(max(x0 - r + (int)threadIdx.x, 0), W - 1);  // this thread's (clamped) input column
  const uint8_t* col = in + (int64_t)f * in_fs + 3LL * xc;
  const int64_t pitch = 3LL * W;
  auto feat = [&](int y, double& g, double& p) {
    const uint8_t* px = col + (int64_t)min(max(y, 0), H - 1) * pitch;
    const uint32_t R = px[0], G = px[1], B = px[2];
    g = guide_t(T, R, G, B);
    p = T.t[min(min(R, G), B)];
  };
  // vertical window sums for output row y0: rows y0-r .. y0+r (clamped)
  double sg = 0.0, sp = 0.0, sgp = 0.0, sgg = 0.0;
  for (int d = -r; d <= r; ++d) {
    double g, p;
    feat(y0 + d, g, p);
    sg = __dadd_rn(sg, g);
    sp = __dadd_rn(sp, p);
    sgp = __dadd_rn(sgp, __dmul_rn(g, p));
    sgg = __dadd_rn(sgg, __dmul_rn(g, g));
  }
  const double kk = (double)(2 * r + 1) * (double)(2 * r + 1);
  const double rkk = __drcp_rn(kk);
  const int j = (int)threadIdx.x - r;  // output column index within the strip (valid if 0 <= j < sw)
  const int xo = x0 + j;
  const bool active = j >= 0 && j < sw && xo < W;
  const int hi = j + 2 * r + 1, lo = j;
  int buf = 0;
  for (int y = y0; y < y1; ++y, buf ^= 1) {
    if (y > y0) {
      double g, p, g2, p2;
      feat(y + r, g, p);
      feat(y - r - 1, g2, p2);
      sg = __dsub_rn(__dadd_rn(sg, g), g2);
      sp = __dsub_rn(__dadd_rn(sp, p), p2);
      sgp = __dsub_rn(__dadd_rn(sgp, __dmul_rn(g, p)), __dmul_rn(g2, p2));
      sgg = __dsub_rn(__dadd_rn(sgg, __dmul_rn(g, g)), __dmul_rn(g2, g2));
    }
    double v[4] = {sg, sp, sgp, sgg};
    cta_prefix<4>(v, wt[buf]);
#pragma unroll
    for (int q = 0; q < 4; ++q) pre[buf][q][threadIdx.x + 1] = v[q];
    __syncthreads();
    if (active) {
      // window over input columns [j, j + 2r] of the strip = prefix[j+2r+1] - prefix[j]
      const double mi = div_rb(__dsub_rn(pre[buf][0][hi], pre[buf][0][lo]), kk, rkk);
      const double mp = div_rb(__dsub_rn(pre[buf][1][hi], pre[buf][1][lo]), kk, rkk);
      const double cip = div_rb(__dsub_rn(pre[buf][2][hi], pre[buf][2][lo]), kk, rkk);
      const double cii = div_rb(__dsub_rn(pre[buf][3][hi], pre[buf][3][lo]), kk, rkk);
      const double var = __dsub_rn(cii, __dmul_rn(mi, mi));
      const double cov = __dsub_rn(cip, __dmul_rn(mi, mp));
      const double av = __ddiv_rn(cov, __dadd_rn(var, eps));
      const int64_t o = (int64_t)f * H * W + (int64_t)y * W + xo;
      a_out[o] = av;
      b_out[o] = __dsub_rn(mp, __dmul_rn(av, mi));
    }
    // no trailing barrier: the next row uses the other pre/wt buffer, and the
    // barrier inside its cta_prefix orders this row's reads before buf is reused
  }
}

// ---------------------------------------------------------------- pass 2 ----
// clip(((v/255 - A) / t) + A, 0, 1) with the division done as div_rb(., t, RN(1/t)).
__device__ __forceinline__ double recover_x(double x, double A, double t, double rt) {
  return fmin(fmax(__dadd_rn(div_rb(__dsub_rn(x, A), t, rt), A), 0.0), 1.0);
}

// MODE 0: write output bytes (no balance).  MODE 1: write t~ and per-CTA channel
// sums of the gamma values (gray-world balance follows in k_gf_apply).
template <int MODE>
__global__ void __launch_bounds__(kCols)
k_gf_pass2(const uint8_t* __restrict__ in, int64_t in_fs, int H, int W, int r, int seg,
           const double* __restrict__ a_in,
           const double* __restrict__ b_in, const double* __restrict__ airlight, double t_min,
           const double* __restrict__ thr, double inv_gamma, int gamma_is_one, uint8_t* __restrict__ out,
           int64_t out_fs, double* __restrict__ t_out, double* __restrict__ part) {
  __shared__ GuideTables T;  // wr/wg/wb for the guide; t[] holds v/255 here
  __shared__ double sA[3], s_thr[256];
  __shared__ double pre[2][2][kCols + 1];
  __shared__ double wt[2][2][kCols / 32];
  const int f = blockIdx.z;
  const int sw = kCols - 2 * r;
  const int x0 = blockIdx.x * sw;
  const int y0 = blockIdx.y * seg;
  const int y1 = min(H, y0 + seg);
  {
    const int v = threadIdx.x;
    const double x = u8f(v);
    T.wr[v] = __dmul_rn(0.299, x);
    T.wg[v] = __dmul_rn(0.587, x);
    T.wb[v] = __dmul_rn(0.114, x);
    T.t[v] = x;
    s_thr[v] = thr[v];
  }
  if (threadIdx.x < 3) sA[threadIdx.x] = airlight[3 * f + threadIdx.x];
  if (threadIdx.x < 4) pre[threadIdx.x >> 1][threadIdx.x & 1][0] = 0.0;
  __syncthreads();
  const int xc = min(max(x0 - r + (int)threadIdx.x, 0), W - 1);
  const int64_t fo = (int64_t)f * H * W;
  auto ab = [&](int y, double& a, double& b) {
    const int64_t o = fo + (int64_t)min(max(y, 0), H - 1) * W + xc;
    a = a_in[o];
    b = b_in[o];
  };
  double sa = 0.0, sb = 0.0;
  for (int d = -r; d <= r; ++d) {
    double a, b;
    ab(y0 + d, a, b);
    sa = __dadd_rn(sa, a);
    sb = __dadd_rn(sb, b);
  }
  const double kk = (double)(2 * r + 1) * (double)(2 * r + 1);
  const double rkk = __drcp_rn(kk);
  const int j = (int)threadIdx.x - r;
  const int xo = x0 + j;
  const bool active = j >= 0 && j < sw && xo < W;
  const int hi = j + 2 * r + 1, lo = j;
  const uint8_t* frame = in + (int64_t)f * in_fs;
  const double A0 = sA[0], A1 = sA[1], A2 = sA[2];
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  int buf = 0;
  for (int y = y0; y < y1; ++y, buf ^= 1) {
    if (y > y0) {
      double a, b, a2, b2;
      ab(y + r, a, b);
      ab(y - r - 1, a2, b2);
      sa = __dsub_rn(__dadd_rn(sa, a), a2);
      sb = __dsub_rn(__dadd_rn(sb, b), b2);
    }
    double v[2] = {sa, sb};
    cta_prefix<2>(v, wt[buf]);
    pre[buf][0][threadIdx.x + 1] = v[0];
    pre[buf][1][threadIdx.x + 1] = v[1];
    __syncthreads();
    if (active) {
      const double ma = div_rb(__dsub_rn(pre[buf][0][hi], pre[buf][0][lo]), kk, rkk);
      const double mb = div_rb(__dsub_rn(pre[buf][1][hi], pre[buf][1][lo]), kk, rkk);
      const uint8_t* px = frame + ((int64_t)y * W + xo) * 3;
      const uint32_t R = px[0], G = px[1], B = px[2];
      const double g = guide_t(T, R, G, B);
      double t = fmin(fmax(__dadd_rn(__dmul_rn(ma, g), mb), 0.0), 1.0);
      t = fmax(t, t_min);  // pipeline.py:203
      const double rt = __drcp_rn(t);
      const double x0v = recover_x(T.t[R], A0, t, rt), x1v = recover_x(T.t[G], A1, t, rt),
                   x2v = recover_x(T.t[B], A2, t, rt);
      if (MODE == 0) {
        uint8_t* o = out + (int64_t)f * out_fs + ((int64_t)y * W + xo) * 3;
        o[0] = (uint8_t)quantize_thr(x0v, s_thr);
        o[1] = (uint8_t)quantize_thr(x1v, s_thr);
        o[2] = (uint8_t)quantize_thr(x2v, s_thr);
      } else {
        t_out[fo + (int64_t)y * W + xo] = t;
        if (gamma_is_one) {
          acc0 = __dadd_rn(acc0, x0v);
          acc1 = __dadd_rn(acc1, x1v);
          acc2 = __dadd_rn(acc2, x2v);
        } else {
          acc0 = __dadd_rn(acc0, fmin(fmax(pow(x0v, inv_gamma), 0.0), 1.0));
          acc1 = __dadd_rn(acc1, fmin(fmax(pow(x1v, inv_gamma), 0.0), 1.0));
          acc2 = __dadd_rn(acc2, fmin(fmax(pow(x2v, inv_gamma), 0.0), 1.0));
        }
      }
    }
  }
  if (MODE == 1) {
    double v3[3] = {acc0, acc1, acc2};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < 3; ++c) v3[c] = __dadd_rn(v3[c], __shfl_xor_sync(0xffffffffu, v3[c], o));
    __syncthreads();  // pre[][] is reused as the cross-warp buffer
    double* red = &pre[0][0][0];
    if ((threadIdx.x & 31) == 0)
      for (int c = 0; c < 3; ++c) red[c * 8 + (threadIdx.x >> 5)] = v3[c];
    __syncthreads();
    if (threadIdx.x < 3) {
      double s = 0.0;
      for (int w = 0; w < kCols / 32; ++w) s = __dadd_rn(s, red[threadIdx.x * 8 + w]);
      const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
      part[((int64_t)f * gridDim.x * gridDim.y + cta) * 3 + threadIdx.x] = s;
    }
  }
}

// gray-world apply: gains from the per-CTA partial sums, then out = u8(clip(g * gain)).
__global__ void __launch_bounds__(256)
k_gf_apply(const uint8_t* __restrict__ in, int64_t in_fs, int64_t npx, const double* __restrict__ t_in,
           const double* __restrict__ airlight, double inv_gamma, int gamma_is_one, const double* __restrict__ part,
           int nparts, uint8_t* __restrict__ out, int64_t out_fs) {
  __shared__ double s_gain[3], s_f[256];
  __shared__ int s_copy;
  const int f = blockIdx.y;
  s_f[threadIdx.x] = u8f(threadIdx.x);
  if (threadIdx.x == 0) {
    double m[3];
    for (int c = 0; c < 3; ++c) {
      double s = 0.0;
      for (int b = 0; b < nparts; ++b) s = __dadd_rn(s, part[((int64_t)f * nparts + b) * 3 + c]);
      m[c] = __ddiv_rn(s, (double)npx);
    }
    const bool degenerate = fmin(fmin(m[0], m[1]), m[2]) < 1e-6;
    const double mm = __ddiv_rn(__dadd_rn(__dadd_rn(m[0], m[1]), m[2]), 3.0);
    for (int c = 0; c < 3; ++c) s_gain[c] = degenerate ? 1.0 : fmin(fmax(__ddiv_rn(mm, m[c]), 0.5), 2.0);
    s_copy = degenerate;
  }
  __syncthreads();
  const double A0 = airlight[3 * f], A1 = airlight[3 * f + 1], A2 = airlight[3 * f + 2];
  const uint8_t* fi = in + (int64_t)f * in_fs;
  uint8_t* fo = out + (int64_t)f * out_fs;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
    const double t = t_in[(int64_t)f * npx + p];
    const double rt = __drcp_rn(t);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double x = recover_x(s_f[fi[3 * p + c]], c == 0 ? A0 : (c == 1 ? A1 : A2), t, rt);
      const double g = gamma_is_one ? x : fmin(fmax(pow(x, inv_gamma), 0.0), 1.0);
      fo[3 * p + c] = (uint8_t)quantize_unit(s_copy ? g : fmin(fmax(__dmul_rn(g, s_gain[c]), 0.0), 1.0));
    }
  }
}

}  // namespace

// Rows per CTA segment: long segments amortise the 2r+1-row warm-up of the
// sliding sums, short ones give small batches enough CTAs (>= ~4 per SM).
int guided_seg_rows(int H, int W, int r, int n) {
  const int sw = kCols - 2 * r;
  const int64_t strips = (int64_t)((W + sw - 1) / sw) * n;
  const int64_t want = 8 * 148;  // ~2 waves at 4 resident CTAs per SM
  int64_t segs = std::max<int64_t>(1, (want + strips - 1) / strips);
  int seg = (int)((H + segs - 1) / segs);
  seg = std::max(seg, std::min(H, std::max(16, r)));  // the 2r+1-row warm-up is cheap next to a row
  return std::min(seg, 1024);
}

// Frames per chunk so the fp64 a/b (+t~) scratch stays within ~4 GB.
int guided_chunk(int n, int H, int W, bool balance) {
  const double per = (balance ? 24.0 : 16.0) * (double)H * W;
  return (int)std::max(1.0, std::min((double)n, 4.0e9 / per));
}

size_t guided_ws_bytes(int n, int H, int W, int r, bool balance) {
  const int64_t npx = (int64_t)H * W;
  const int c = guided_chunk(n, H, W, balance);
  const int sw = kCols - 2 * r;
  const int seg = guided_seg_rows(H, W, r, c);
  const int64_t parts = (int64_t)((W + sw - 1) / sw) * ((H + seg - 1) / seg);
  size_t b = 16ull * npx * c;                             // a, b
  if (balance) b += 8ull * npx * c + 24ull * parts * c;   // t~, partial sums
  return b;
}

cudaError_t guided_recover_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, double eps,
                              const double* airlight, double omega, double t_min, const double* thr, double gamma,
                              bool balance, uint8_t* out, int64_t out_fs, void* ws, cudaStream_t st) {
  if (r < 1 || 2 * r >= kCols) return cudaErrorInvalidValue;
  const int64_t npx = (int64_t)H * W;
  const int sw = kCols - 2 * r;
  const int chunk = guided_chunk(n, H, W, balance);
  const double inv_g = 1.0 / gamma;
  const int g1 = gamma == 1.0 ? 1 : 0;
  for (int f0 = 0; f0 < n; f0 += chunk) {
    const int c = std::min(chunk, n - f0);
    const int seg = guided_seg_rows(H, W, r, c);
    dim3 grid((W + sw - 1) / sw, (H + seg - 1) / seg, c);
    const uint8_t* fin = in + (int64_t)f0 * in_fs;
    uint8_t* fout = out + (int64_t)f0 * out_fs;
    const double* fA = airlight + 3 * f0;
    double* a = static_cast<double*>(ws);
    double* b = a + npx * c;
    k_gf_pass1<<<grid, kCols, 0, st>>>(fin, in_fs, H, W, r, seg, eps, fA, omega, t_min, a, b);
    if (!balance) {
      k_gf_pass2<0><<<grid, kCols, 0, st>>>(fin, in_fs, H, W, r, seg, a, b, fA, t_min, thr, inv_g, g1, fout, out_fs,
                                            nullptr, nullptr);
    } else {
      double* t = b + npx * c;
      double* part = t + npx * c;
      k_gf_pass2<1><<<grid, kCols, 0, st>>>(fin, in_fs, H, W, r, seg, a, b, fA, t_min, thr, inv_g, g1, fout, out_fs,
                                            t, part);
      const int nparts = grid.x * grid.y;
      dim3 g2((unsigned)std::min<int64_t>(4096, (npx + 255) / 256), c);
      k_gf_apply<<<g2, 256, 0, st>>>(fin, in_fs, npx, t, fA, inv_g, g1, part, nparts, fout, out_fs);
    }
  }
  return cudaGetLastError();
}

}  // namespace dhz
