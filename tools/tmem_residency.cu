// Residency of tcgen05 kernels: what the occupancy API answers vs what the
// hardware keeps resident.  Build + run (one GPU):
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_residency tools/tmem_residency.cu && /tmp/tmem_residency
// Output recorded in profiles/r2_tmem_residency.txt; see DESIGN.md "Occupancy of tcgen05 kernels".
#include <cstdio>
#include <cstdint>
extern __shared__ char smem[];
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
template <bool kT>
__global__ void __launch_bounds__(128) k_probe(unsigned* cnt, int* ok, int* maxco) {
  __shared__ uint32_t taddr;
  if (kT && threadIdx.x < 32) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&taddr));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" :: "r"(a));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  smem[threadIdx.x] = 1;
  if (threadIdx.x == 0) {
    unsigned v = atomicAdd(cnt, 1u) + 1;
    uint64_t t0 = gtime();
    while (v < gridDim.x && gtime() - t0 < 20000000ull) { v = atomicAdd(cnt, 0u); __nanosleep(200); }
    atomicMax(maxco, (int)v);
    if (v >= gridDim.x) atomicAdd(ok, 1);
  }
  __syncthreads();
  if (kT && threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" :: "r"(taddr));
}
int main() {
  for (int s : {0, 16384, 50240, 60000}) {
    cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    int a = -1, b = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, k_probe<false>, 128, s);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_probe<true>, 128, s);
    printf("occupancy API, %d B dynamic smem: plain %d, with tcgen05.alloc %d\n", s, a, b);
  }
  unsigned* cnt; int *ok, *mx;
  cudaMalloc(&cnt, 4); cudaMalloc(&ok, 4); cudaMalloc(&mx, 4);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  for (int per : {1, 2, 3, 4}) for (int t = 0; t < 2; ++t) {
    cudaMemset(cnt, 0, 4); cudaMemset(ok, 0, 4); cudaMemset(mx, 0, 4);
    int g = per * sms;
    if (t) k_probe<true><<<g, 128, 50240>>>(cnt, ok, mx); else k_probe<false><<<g, 128, 50240>>>(cnt, ok, mx);
    cudaError_t e = cudaDeviceSynchronize();
    int o = 0, m = 0; cudaMemcpy(&o, ok, 4, cudaMemcpyDeviceToHost); cudaMemcpy(&m, mx, 4, cudaMemcpyDeviceToHost);
    printf("tmem %d per_sm %d grid %d: all-arrived %d of %d, max co-resident %d (%s)\n", t, per, g, o, g, m, cudaGetErrorString(e));
  }
}
