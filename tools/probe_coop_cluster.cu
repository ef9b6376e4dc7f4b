// Probe: a 2-CTA-cluster kernel with a software grid barrier, launched with the
// cooperative attribute (+ PDL), eagerly and inside a CUDA graph, while a
// second kernel holds part of the SMs on another stream. Answers whether the
// driver accepts cooperative + cluster + PDL together, and what it costs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        -o tools/libprobe_coop_cluster.so tools/probe_coop_cluster.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

__device__ unsigned g_cnt, g_gen;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    barrier_kernel(int* out, long long spin_ns) {
  extern __shared__ unsigned char sm[];
  sm[threadIdx.x] = (unsigned char)threadIdx.x;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  // some work before the barrier so CTAs arrive at different times
  if (blockIdx.x % 7 == 0) {
    unsigned long long t;
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)spin_ns);
  }
  out[blockIdx.x] = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned my;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(my) : "l"(&g_gen) : "memory");
    __threadfence();
    if (atomicAdd(&g_cnt, 1u) == gridDim.x - 1) {
      atomicExch(&g_cnt, 0u);
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&g_gen), "r"(my + 1) : "memory");
    } else {
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&g_gen) : "memory");
      } while (g == my);
    }
  }
  __syncthreads();
  // after the barrier every CTA's flag must be visible
  if (threadIdx.x == 0) {
    int s = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) s += ((volatile int*)out)[b];
    out[gridDim.x + blockIdx.x] = s;
  }
}

__global__ void busy_kernel(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)ns);
}

static cudaError_t launch(int clusters, size_t smem, int* out, long long spin, cudaStream_t st, int coop, int pdl) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (coop) {
    at[n].id = cudaLaunchAttributeCooperative;
    at[n].val.cooperative = 1;
    ++n;
  }
  if (pdl) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, barrier_kernel, out, spin);
}

extern "C" int probe_run(int clusters, int smem_kb, int coop, int pdl, int graph, int busy_blocks, int* out,
                         float* ms) {
  size_t smem = (size_t)smem_kb * 1024;
  cudaFuncSetAttribute(barrier_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaMemset(out, 0, sizeof(int) * 4 * clusters);
  cudaDeviceSynchronize();
  cudaError_t err = cudaSuccess;
  cudaGraphExec_t ge = nullptr;
  cudaGraph_t g = nullptr;
  if (graph) {
    cudaStreamBeginCapture(a, cudaStreamCaptureModeGlobal);
    err = launch(clusters, smem, out, 20000, a, coop, pdl);
    cudaError_t e2 = cudaStreamEndCapture(a, &g);
    if (err == cudaSuccess) err = e2;
    if (err == cudaSuccess) err = cudaGraphInstantiate(&ge, g, 0);
    if (err != cudaSuccess) {
      printf("capture: %s\n", cudaGetErrorString(err));
      cudaGetLastError();
      return (int)err;
    }
  }
  if (busy_blocks) busy_kernel<<<busy_blocks, 128, 0, b>>>(2000000);  // 2 ms on some SMs
  cudaEventRecord(e0, a);
  if (graph) err = cudaGraphLaunch(ge, a);
  else err = launch(clusters, smem, out, 20000, a, coop, pdl);
  cudaEventRecord(e1, a);
  if (err != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(err));
  cudaError_t se = cudaDeviceSynchronize();
  if (se != cudaSuccess) printf("sync: %s\n", cudaGetErrorString(se));
  cudaEventElapsedTime(ms, e0, e1);
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  return err != cudaSuccess ? (int)err : (int)se;
}

extern "C" int probe_max_clusters(int smem_kb) {
  size_t smem = (size_t)smem_kb * 1024;
  cudaFuncSetAttribute(barrier_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(296);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  cudaOccupancyMaxActiveClusters(&n, (void*)barrier_kernel, &cfg);
  return n;
}
