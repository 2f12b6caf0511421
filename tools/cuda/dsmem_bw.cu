// dsmem_bw.cu — distributed shared memory throughput of a 2-CTA cluster on
// B200: remote loads / stores of 8- and 16-byte elements vs local, per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bw dsmem_bw.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int VEC, bool REMOTE, bool STORE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(352, 1) k_bw(double* out, int iters) {
    extern __shared__ double sm[];
    constexpr int NE = 20000;  // doubles per CTA buffer (160 KB)
    cg::cluster_group cl = cg::this_cluster();
    const unsigned peer = cl.block_rank() ^ 1u;
    for (int k = threadIdx.x; k < NE; k += blockDim.x) sm[k] = k;
    cl.sync();
    double* buf = REMOTE ? cl.map_shared_rank(sm, peer) : sm;
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        for (int k = threadIdx.x * VEC; k + VEC <= NE; k += blockDim.x * VEC) {
            if (VEC == 2) {
                double2* p = reinterpret_cast<double2*>(buf + k);
                if (STORE) *p = make_double2(acc, acc + 1.0);
                else {
                    const double2 v = *p;
                    acc += v.x + v.y;
                }
            } else {
                if (STORE) buf[k] = acc;
                else acc += buf[k];
            }
        }
        if (STORE) acc += 1.0;
    }
    cl.sync();
    if (acc == -1.0) out[0] = acc;
}

template <int VEC, bool REMOTE, bool STORE>
void run(const char* name, double* out) {
    auto k = k_bw<VEC, REMOTE, STORE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160000);
    const int iters = 200;
    k<<<148, 352, 160000>>>(out, 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 352, 160000>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 148.0 * 20000 * 8 * iters;  // per direction, all SMs
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-22s %8.3f ms  %8.1f GB/s total  %6.1f B/cycle/SM (err %s)\n", name, ms, bytes / (ms * 1e-3) / 1e9,
           bytes / 148.0 / cyc, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    run<1, false, false>("local load 8B", out);
    run<2, false, false>("local load 16B", out);
    run<1, true, false>("remote load 8B", out);
    run<2, true, false>("remote load 16B", out);
    run<1, false, true>("local store 8B", out);
    run<2, false, true>("local store 16B", out);
    run<1, true, true>("remote store 8B", out);
    run<2, true, true>("remote store 16B", out);
    return 0;
}
