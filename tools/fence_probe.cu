// fence_probe.cu -- latency of system-scope fences under different loads
// (dev tool).  One process, GPU 0 (and GPU 1 for the NVLink case):
//   mode 0: idle GPU
//   mode 1: every other SM streams HBM copies
//   mode 2: every other SM streams stores into GPU 1's memory (peer access)
//   mode 3: like 2, and the probing warp's own SM also streams peer stores
// The probe warp (on the SM that gets CTA 0) times fence.acq_rel.sys,
// fence.acq_rel.gpu and st.release.sys with clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o fence_probe tools/fence_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ volatile int g_stop;

__global__ void probe(float* src, float* dst, size_t n, int mode, unsigned long long* out, uint32_t* flag) {
  const bool prober = blockIdx.x == 0 && threadIdx.x < 32;
  if (prober) {
    if (threadIdx.x == 0) {
      // warm up / let the streamers start
      unsigned long long t0 = clock64();
      while (clock64() - t0 < 200000) {
      }
      unsigned long long a = 0, b = 0, c = 0;
      const int reps = 64;
      for (int r = 0; r < reps; ++r) {
        unsigned long long s = clock64();
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        unsigned long long e = clock64();
        a += e - s;
        s = clock64();
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        e = clock64();
        b += e - s;
        s = clock64();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(r) : "memory");
        e = clock64();
        c += e - s;
      }
      out[0] = a / reps;
      out[1] = b / reps;
      out[2] = c / reps;
      g_stop = 1;
    }
    return;
  }
  if (mode == 0 || (blockIdx.x == 0 && mode != 3)) return;
  // streamers: grid-stride copies until the prober is done
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (int it = 0; it < 1000 && !g_stop; ++it)
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
      reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
}

int main() {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  const size_t n = (size_t)64 << 20;  // float4s = 1 GiB
  float *src, *dst_local, *dst_peer = nullptr;
  unsigned long long* out;
  uint32_t* flag;
  cudaSetDevice(0);
  cudaMalloc(&src, n * 16);
  cudaMalloc(&dst_local, n * 16);
  cudaMallocManaged(&out, 64);
  cudaMalloc(&flag, 64);
  if (ndev > 1) {
    cudaDeviceEnablePeerAccess(1, 0);
    cudaSetDevice(1);
    cudaMalloc(&dst_peer, n * 16);
    cudaSetDevice(0);
  }
  const char* names[] = {"idle", "HBM stream on other SMs", "peer stores on other SMs", "peer stores on all SMs"};
  for (int mode = 0; mode < 4; ++mode) {
    if (mode >= 2 && !dst_peer) break;
    int zero = 0;
    cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    probe<<<148, 512>>>(src, mode >= 2 ? dst_peer : dst_local, n, mode, out, flag);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    printf("%-28s fence.acq_rel.sys %7llu cyc  fence.acq_rel.gpu %7llu cyc  st.release.sys %7llu cyc\n", names[mode],
           out[0], out[1], out[2]);
  }
  return 0;
}
