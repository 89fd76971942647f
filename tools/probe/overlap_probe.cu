// Feasibility probe: do K1 (dark, ALU-bound) and K6 (LUT apply, LSU-bound) overlap
// when they run concurrently on two streams over independent frame sets?
// Build: see tools/probe/build.sh.  Prints K1 alone, K6 alone, both concurrently.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2512_16609_b200/csrc/dhz_internal.h"
#include "../../paper_2512_16609_b200/csrc/dhz_common.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  const int n = 300, H = 1080, W = 1920;
  const int64_t fs = 3LL * H * W, npx = (int64_t)H * W;
  uint8_t *inA, *inB, *out, *dark, *lut;
  uint32_t *fmax, *bmax;
  CK(cudaMalloc(&inA, fs * n));
  CK(cudaMalloc(&inB, fs * n));
  CK(cudaMalloc(&out, fs * n));
  CK(cudaMalloc(&dark, npx * n));
  CK(cudaMalloc(&lut, (size_t)dhz::kLutFrame * n));
  CK(cudaMalloc(&fmax, 4 * n));
  const int nb = (H + 15) / 16, ntx = (W + 479) / 480;
  CK(cudaMalloc(&bmax, 4LL * n * nb * ntx));
  CK(cudaMemset(inA, 120, fs * n));
  CK(cudaMemset(inB, 90, fs * n));
  CK(cudaMemset(lut, 7, (size_t)dhz::kLutFrame * n));
  // random-ish content
  {
    uint8_t* h = (uint8_t*)malloc(fs * 8);
    uint32_t s = 12345;
    for (int64_t i = 0; i < fs * 8; ++i) { s = s * 1664525u + 1013904223u; h[i] = 80 + ((s >> 24) % 100); }
    for (int f = 0; f < n; f += 8) {
      CK(cudaMemcpy(inA + f * fs, h, fs * std::min(8, n - f), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(inB + f * fs, h, fs * std::min(8, n - f), cudaMemcpyHostToDevice));
    }
    free(h);
  }
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, e2, e3;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
  auto k1 = [&](cudaStream_t st) { return dhz::dark_u8(inA, fs, n, H, W, 7, dark, npx, fmax, bmax, st); };
  auto k6 = [&](cudaStream_t st) { return dhz::recover_lut_u8(inB, fs, n, H, W, lut, out, fs, st); };
  for (int w = 0; w < 3; ++w) { k1(s1); k6(s1); }
  CK(cudaDeviceSynchronize());
  float t;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, s1); k1(s1); cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1); printf("K1 alone  %.3f ms\n", t);
    cudaEventRecord(e0, s1); k6(s1); cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1); printf("K6 alone  %.3f ms\n", t);
    cudaEventRecord(e0, s1); k1(s1); k6(s1); cudaEventRecord(e1, s1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1); printf("K1;K6     %.3f ms\n", t);
    cudaEventRecord(e0, s1);
    cudaStreamWaitEvent(s2, e0, 0);
    k6(s2);  // persistent K6 first, then K1 fills the rest
    k1(s1);
    cudaEventRecord(e2, s2);
    cudaStreamWaitEvent(s1, e2, 0);
    cudaEventRecord(e1, s1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1); printf("K6 || K1  %.3f ms\n", t);
  }
  CK(cudaGetLastError());
  return 0;
}
