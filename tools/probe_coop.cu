// Probe: does a cooperative launch (grid.sync) work inside CUDA-graph stream capture?
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdio.h>
namespace cg = cooperative_groups;

__global__ void coop_sum(const float* x, float* part, float* out, int n) {
  cg::grid_group grid = cg::this_grid();
  float s = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += x[i];
  __shared__ float red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int k = 0; k < blockDim.x; ++k) t += red[k];
    part[blockIdx.x] = t;
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    float t = 0.f;
    for (int b = 0; b < gridDim.x; ++b) t += part[b];
    out[0] = t;
  }
}

extern "C" int probe_coop(const float* x, float* part, float* out, int n, int blocks, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, coop_sum, x, part, out, n);
  if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
  return (int)e;
}
extern "C" int probe_coop_maxblocks() {
  int nb = 0, dev = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, coop_sum, 256, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return nb * sms;
}
