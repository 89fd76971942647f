// Multi-GPU plumbing of the C ABI (one process, several devices) and the opt-in
// temporal stabilisation of the airlight trace (north_star; NOT reference
// behaviour: SPEC.md:267 lists temporal smoothing as a non-goal).
//
// Frames are independent (reference pipeline.py:257-260), so a batch shards into
// contiguous frame blocks, one per device; the only exchange is the per-frame
// airlight (24 B/frame), all-gathered so every device holds the trace in frame
// order (StreamStats.airlight_trace, pipeline.py:279,308).  Within one process the
// all-gather is a set of peer copies over NVLink ordered by events; across
// processes (torchrun) the host side uses NCCL through torch.distributed.
#include <cstdlib>
#include <new>

#include "../../include/dehaze_b200.h"
#include "dhz_internal.h"

namespace {

constexpr int kMaxDev = 64;

struct Comm {
  int ndev;
  int devs[kMaxDev];
  cudaEvent_t ev[kMaxDev];
};

// A'_f = lam A'_{f-1} + (1 - lam) A_f per channel, A'_-1 = carry (or A'_0 = A_0 without
// one); every product and sum rounded once (no FMA), so the trace is reproducible
// bit for bit by any IEEE double evaluation of the same recurrence.  One thread per
// channel: the recurrence is sequential in f (~10 cycles per frame).
__global__ void k_ema(const double* __restrict__ trace, int n, double lam, const double* __restrict__ carry,
                      double* __restrict__ out) {
  const int c = threadIdx.x;
  if (c >= 3) return;
  const double keep = lam, take = __dsub_rn(1.0, lam);
  double a;
  int f = 0;
  if (carry) {
    a = carry[c];
  } else {
    a = trace[c];
    out[c] = a;
    f = 1;
  }
  for (; f < n; ++f) {
    a = __dadd_rn(__dmul_rn(keep, a), __dmul_rn(take, trace[3 * f + c]));
    out[3 * f + c] = a;
  }
}

int set_dev(int d, const char* where) {
  const cudaError_t e = cudaSetDevice(d);
  return e == cudaSuccess ? DHZ_OK : dhz::abi_cuda_fail(e, where);
}

}  // namespace

extern "C" {

int dhz_ema_airlight(const double* trace, int n, double lam, const double* carry, double* out, void* stream) {
  if (n < 0) return dhz::abi_fail(DHZ_E_INVALID, "n must be >= 0");
  if (!(lam >= 0.0 && lam < 1.0)) return dhz::abi_fail(DHZ_E_INVALID, "lam must lie in [0, 1), got %g", lam);
  if (n == 0) return DHZ_OK;
  if (!trace || !out) return dhz::abi_fail(DHZ_E_INVALID, "NULL array argument");
  k_ema<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(trace, n, lam, carry, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DHZ_OK : dhz::abi_cuda_fail(e, "k_ema");
}

int dhz_comm_init(int ndev, const int* devices, void** comm) {
  if (!comm || !devices) return dhz::abi_fail(DHZ_E_INVALID, "NULL argument");
  if (ndev < 1 || ndev > kMaxDev) return dhz::abi_fail(DHZ_E_INVALID, "ndev must lie in [1, %d]", kMaxDev);
  int prev = 0;
  cudaGetDevice(&prev);
  Comm* c = new (std::nothrow) Comm();
  if (!c) return dhz::abi_fail(DHZ_E_INVALID, "out of host memory");
  c->ndev = ndev;
  int rc = DHZ_OK;
  for (int i = 0; i < ndev && rc == DHZ_OK; ++i) {
    c->devs[i] = devices[i];
    if ((rc = set_dev(devices[i], "dhz_comm_init")) != DHZ_OK) break;
    for (int j = 0; j < ndev; ++j) {  // peer access over NVLink between distinct devices
      if (devices[j] == devices[i]) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, devices[i], devices[j]) == cudaSuccess && can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          rc = dhz::abi_cuda_fail(e, "cudaDeviceEnablePeerAccess");
          break;
        }
        cudaGetLastError();  // clear cudaErrorPeerAccessAlreadyEnabled
      }
    }
    if (rc == DHZ_OK) {
      const cudaError_t e = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) rc = dhz::abi_cuda_fail(e, "cudaEventCreate");
    }
  }
  cudaSetDevice(prev);
  if (rc != DHZ_OK) {
    delete c;
    return rc;
  }
  *comm = c;
  return DHZ_OK;
}

int dhz_comm_destroy(void* comm) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c) return DHZ_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  for (int i = 0; i < c->ndev; ++i) {
    cudaSetDevice(c->devs[i]);
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  }
  cudaSetDevice(prev);
  delete c;
  return DHZ_OK;
}

int dhz_allgather_airlight(void* comm, const double* const* send, const int* counts, double* const* recv,
                           void* const* streams) {
  Comm* c = static_cast<Comm*>(comm);
  if (!c || !send || !counts || !recv || !streams) return dhz::abi_fail(DHZ_E_INVALID, "NULL argument");
  int prev = 0;
  cudaGetDevice(&prev);
  int rc = DHZ_OK;
  for (int s = 0; s < c->ndev && rc == DHZ_OK; ++s) {  // each block is final once its stream gets here
    if (counts[s] < 0) rc = dhz::abi_fail(DHZ_E_INVALID, "negative count");
    else if ((rc = set_dev(c->devs[s], "dhz_allgather_airlight")) == DHZ_OK) {
      const cudaError_t e = cudaEventRecord(c->ev[s], reinterpret_cast<cudaStream_t>(streams[s]));
      if (e != cudaSuccess) rc = dhz::abi_cuda_fail(e, "cudaEventRecord");
    }
  }
  for (int d = 0; d < c->ndev && rc == DHZ_OK; ++d) {
    if ((rc = set_dev(c->devs[d], "dhz_allgather_airlight")) != DHZ_OK) break;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(streams[d]);
    int64_t off = 0;
    for (int s = 0; s < c->ndev; ++s) {
      if (counts[s] > 0) {
        cudaError_t e = cudaStreamWaitEvent(st, c->ev[s], 0);
        if (e == cudaSuccess)
          e = cudaMemcpyPeerAsync(recv[d] + 3 * off, c->devs[d], send[s], c->devs[s], 24ull * counts[s], st);
        if (e != cudaSuccess) {
          rc = dhz::abi_cuda_fail(e, "peer copy");
          break;
        }
      }
      off += counts[s];
    }
  }
  cudaSetDevice(prev);
  return rc;
}

}  // extern "C"
