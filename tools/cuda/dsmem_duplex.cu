// dsmem_duplex.cu — is DSMEM throughput per direction or shared?  2-CTA
// clusters on all SMs; per CTA role: 0 idle, 1 remote loads (x8 in flight),
// 2 remote stores, 3 half the threads load + half store.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_duplex dsmem_duplex.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
constexpr int NE = 20000;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) k(double* out, int iters, int role0, int role1) {
    extern __shared__ double sm[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank(), peer = rank ^ 1u;
    for (int i = threadIdx.x; i < NE; i += blockDim.x) sm[i] = i;
    cl.sync();
    double* rem = cl.map_shared_rank(sm, peer);
    const int role = rank == 0 ? role0 : role1;
    double acc = 0.0;
    const int nt = blockDim.x;
    for (int it = 0; it < iters; ++it) {
        int r = role;
        int tid = threadIdx.x, n = nt;
        if (role == 3) {  // split the CTA
            r = threadIdx.x < nt / 2 ? 1 : 2;
            tid = threadIdx.x % (nt / 2);
            n = nt / 2;
        }
        if (r == 1) {
            for (int i = tid; i + 7 * n < NE; i += 8 * n) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = rem[i + u * n];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += v[u];
            }
        } else if (r == 2) {
            for (int i = tid; i < NE; i += n) rem[(i + 10000) % NE] = acc + i;
            acc += 1.0;
        }
    }
    cl.sync();
    if (acc == -1.0) out[0] = acc;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    const int smem = NE * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const char* nm[] = {"idle", "load", "store", "ld+st"};
    int cases[][2] = {{1, 1}, {1, 0}, {2, 2}, {2, 0}, {1, 2}, {3, 3}, {3, 0}};
    for (auto& c : cases) {
        k<<<148, 384, smem>>>(out, 2, c[0], c[1]);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int iters = 200;
        cudaEventRecord(e0);
        k<<<148, 384, smem>>>(out, iters, c[0], c[1]);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double cyc = ms * 1e-3 * clk * 1e3;
        // bytes moved by one active CTA per iteration: NE * 8
        printf("rank0 %-6s rank1 %-6s  %8.3f ms  %6.1f B/cycle per active CTA (err %s)\n", nm[c[0]], nm[c[1]], ms,
               (double)NE * 8 * iters / cyc, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
