// barrier_lat.cu — cost of one CTA barrier and one 2-CTA cluster barrier
// (barrier.cluster arrive+wait) with 384 threads per CTA, 1 CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_lat barrier_lat.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>  // 0 __syncthreads, 1 cluster barrier (all threads), 2 CTA + cluster (release by warp 0)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) k(long long* out, int iters) {
    extern __shared__ double sm[];
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {
            __syncthreads();
        } else if (MODE == 1) {
            asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            __syncthreads();
            if ((threadIdx.x >> 5) == 0) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            else asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, long long* d, long long* h) {
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    const int iters = 10000;
    k<MODE><<<148, 384, 200000>>>(d, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += h[i];
    printf("%-32s %8.1f cycles per barrier (%s)\n", name, s / 148 / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    long long *d, h[148];
    cudaMalloc(&d, 148 * sizeof(long long));
    run<0>("__syncthreads (384 thr)", d, h);
    run<1>("cluster barrier (all threads)", d, h);
    run<2>("CTA + cluster (warp-0 release)", d, h);
    return 0;
}
