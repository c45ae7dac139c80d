// coresidency_probe.cu -- can a programmatically launched kernel's CTAs share
// SMs with the still-running primary?  (diagnostics for the row-flag path)
// Primary: 148 CTAs x 288 threads, S1 KB dynamic smem, spins ~20 us after
// griddepcontrol.launch_dependents.  Secondary: 148 CTAs x 320 threads, S2 KB
// dynamic smem, optional cluster attribute; records its start time.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(288, 1) primary(unsigned long long* ts, int spin_ns) {
  extern __shared__ unsigned char sm[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const unsigned long long t0 = gt();
  if (threadIdx.x == 0) ts[blockIdx.x * 2] = t0;
  sm[threadIdx.x] = 1;
  while (gt() - t0 < (unsigned long long)spin_ns) {
  }
  if (threadIdx.x == 0) ts[blockIdx.x * 2 + 1] = gt() + sm[5];
}

__global__ void __launch_bounds__(320, 1) secondary(unsigned long long* ts) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0) ts[blockIdx.x] = gt();
  sm[threadIdx.x] = 2;
}

int main(int argc, char** argv) {
  const int s1 = argc > 1 ? atoi(argv[1]) : 45;
  const int s2 = argc > 2 ? atoi(argv[2]) : 137;
  const int cl = argc > 3 ? atoi(argv[3]) : 0;  // secondary cluster dim (0 = no attribute)
  const int carve = argc > 4 ? atoi(argv[4]) : 1;
  unsigned long long *tp, *tsd;
  cudaMalloc(&tp, 148 * 2 * 8);
  cudaMalloc(&tsd, 148 * 8);
  cudaFuncSetAttribute(primary, cudaFuncAttributeMaxDynamicSharedMemorySize, s1 * 1024);
  cudaFuncSetAttribute(secondary, cudaFuncAttributeMaxDynamicSharedMemorySize, s2 * 1024);
  if (carve) {
    cudaFuncSetAttribute(primary, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(secondary, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  for (int rep = 0; rep < 3; ++rep) {
    primary<<<148, 288, s1 * 1024>>>(tp, 20000);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = s2 * 1024;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (cl > 0) {
      attr[na].id = cudaLaunchAttributeClusterDimension;
      attr[na].val.clusterDim.x = cl;
      attr[na].val.clusterDim.y = 1;
      attr[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, secondary, tsd);
    cudaDeviceSynchronize();
    if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
  }
  unsigned long long hp[296], hs[148];
  cudaMemcpy(hp, tp, sizeof(hp), cudaMemcpyDeviceToHost);
  cudaMemcpy(hs, tsd, sizeof(hs), cudaMemcpyDeviceToHost);
  unsigned long long p0 = ~0ull, pend = 0, s0 = ~0ull, smax = 0;
  for (int i = 0; i < 148; ++i) {
    p0 = hp[2 * i] < p0 ? hp[2 * i] : p0;
    pend = hp[2 * i + 1] > pend ? hp[2 * i + 1] : pend;
    s0 = hs[i] < s0 ? hs[i] : s0;
    smax = hs[i] > smax ? hs[i] : smax;
  }
  int early = 0;
  for (int i = 0; i < 148; ++i) early += hs[i] < pend;
  printf("smem %d+%d KB cluster=%d carve=%d: primary %.2f us long; secondary start %.2f..%.2f us; "
         "%d/148 CTAs started while the primary ran\n",
         s1, s2, cl, carve, (pend - p0) / 1e3, ((double)s0 - p0) / 1e3, ((double)smax - p0) / 1e3,
         early);
  return 0;
}
