// exchange.cu — C1/C2: the in-box AFD exchange over NVLink 5 / NVSwitch.
//
// StepMesh analogue (pre-registered tensors, CPU-posted,
// zero SM): buffers are registered once (CUDA IPC handles), every transfer is
// a copy-engine DMA over NVLink enqueued on a stream (no kernel, no SM), and
// readiness travels as 32-bit sequence flags written with stream memory
// operations (cuStreamWriteValue32 into the peer's flag word,
// cuStreamWaitValue32 on the local one) — no host round trip per message.
// Transfers are PULLS: the producer finishes its buffer locally, then raises
// the consumer's flag (the write-value op fences prior stream work); the
// consumer waits on its local flag and DMA-reads the producer's buffer.
// A->F moves fp8 tokens + scales + top-k metadata, F->A moves bf16 partials
// (ffn_net_bytes = (1+2)*H*T, moeplan.cpp:17-20); the attention side then
// reduces the EP partials and adds the residual.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "afdk_internal.h"

namespace afdk {

namespace {

using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WriteValueFn g_write = nullptr;
WaitValueFn g_wait = nullptr;

bool load_memops() {
  if (g_write && g_wait) return true;
  void* fw = nullptr;
  void* fa = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fw, cudaEnableDefault, &q) != cudaSuccess || !fw) return false;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fa, cudaEnableDefault, &q) != cudaSuccess || !fa) return false;
  g_write = reinterpret_cast<WriteValueFn>(fw);
  g_wait = reinterpret_cast<WaitValueFn>(fa);
  return true;
}

// out = base + sum_i partial_i   (bf16 in/out, fp32 sum in fixed order)
__global__ void add_partials_kernel(const __nv_bfloat16* __restrict__ base, const __nv_bfloat16* const* parts,
                                    int n, size_t count, __nv_bfloat16* __restrict__ out) {
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i >= count) return;
  float acc[8];
  {
    const uint4 b = base ? *reinterpret_cast<const uint4*>(base + i) : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(pb[q]);
      acc[2 * q] = f.x;
      acc[2 * q + 1] = f.y;
    }
  }
  for (int p = 0; p < n; ++p) {
    const uint4 v = *reinterpret_cast<const uint4*>(parts[p] + i);
    const __nv_bfloat162* pv = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(pv[q]);
      acc[2 * q] += f.x;
      acc[2 * q + 1] += f.y;
    }
  }
  uint4 o;
  __nv_bfloat162* po = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
  for (int q = 0; q < 4; ++q) po[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
  *reinterpret_cast<uint4*>(out + i) = o;
}

}  // namespace

bool exchange_available() { return load_memops(); }

cudaError_t exchange_signal(uint32_t* flag, uint32_t value, cudaStream_t s) {
  if (!load_memops()) return cudaErrorNotSupported;
  return g_write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value, 0) == CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorLaunchFailure;
}

cudaError_t exchange_wait(const uint32_t* flag, uint32_t value, cudaStream_t s) {
  if (!load_memops()) return cudaErrorNotSupported;
  return g_wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value,
                CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorLaunchFailure;
}

cudaError_t add_partials_launch(const void* base, const void* const* parts_dev, int n, size_t count, void* out,
                                cudaStream_t s) {
  const size_t threads = (count + 7) / 8;
  add_partials_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
      static_cast<const __nv_bfloat16*>(base), reinterpret_cast<const __nv_bfloat16* const*>(parts_dev), n, count,
      static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

}  // namespace afdk
