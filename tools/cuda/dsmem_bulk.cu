// dsmem_bulk.cu — DSMEM throughput of a 2-CTA cluster on B200, three ways:
// per-thread remote loads with 8 independent loads in flight, per-thread
// remote stores, and bulk async copies (cp.async.bulk shared::cta ->
// shared::cluster, the TMA engine) of contiguous regions into the peer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bulk dsmem_bulk.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int NE = 12800;  // doubles per half buffer (100 KB); two halves per CTA

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>  // 0 remote load x8, 1 remote store, 2 bulk push, 3 local load x8
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(352, 1) k_bw(double* out, int iters, int chunk) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) unsigned long long bar;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned peer = cl.block_rank() ^ 1u;
    for (int k = threadIdx.x; k < 2 * NE; k += blockDim.x) sm[k] = k;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    cl.sync();
    double acc = 0.0;
    if (MODE == 2) {
        // each CTA pushes its first half into the peer's second half, in `chunk`-byte copies
        unsigned phase = 0;
        const uint32_t bytes = NE * 8;
        for (int it = 0; it < iters; ++it) {
            if (threadIdx.x == 0) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(bytes));
            }
            cl.sync();  // every CTA armed its barrier before any copy lands
            if (threadIdx.x < 32) {
                const uint32_t nch = bytes / chunk;
                for (uint32_t c = threadIdx.x; c < nch; c += 32) {
                    const uint32_t src = s32(sm) + c * chunk;
                    uint32_t dst = s32(sm + NE) + c * chunk, rbar = s32(&bar), rdst;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(dst), "r"(peer));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(rbar), "r"(peer));
                    asm volatile(
                        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            rdst),
                        "r"(src), "r"(chunk), "r"(rbar)
                        : "memory");
                }
            }
            asm volatile(
                "{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
                    s32(&bar)),
                "r"(phase));
            phase ^= 1u;
        }
        acc = sm[NE + threadIdx.x];
    } else {
        double* buf = (MODE == 3) ? sm : cl.map_shared_rank(sm, peer);
        for (int it = 0; it < iters; ++it) {
            if (MODE == 1) {
                for (int k = threadIdx.x; k < NE; k += blockDim.x) buf[k] = acc + k;
                acc += 1.0;
            } else {
                for (int k = threadIdx.x; k + 7 * 352 < NE; k += 8 * 352) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = buf[k + u * 352];
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc += v[u];
                }
            }
        }
    }
    cl.sync();
    if (acc == -1.0) out[0] = acc;
}

template <int MODE>
void run(const char* name, double* out, int chunk = 0) {
    auto k = k_bw<MODE>;
    const int smem = 2 * NE * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 400;
    k<<<148, 352, smem>>>(out, 2, chunk ? chunk : 4096);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<148, 352, smem>>>(out, iters, chunk ? chunk : 4096);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 148.0 * NE * 8 * iters;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-28s chunk %6d  %8.3f ms  %6.1f B/cycle/SM (err %s)\n", name, chunk, ms, bytes / 148.0 / cyc,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    run<3>("local load x8", out);
    run<0>("remote load x8", out);
    run<1>("remote store", out);
    for (int c : {1024, 4096, 12800, 25600, 51200}) run<2>("bulk push (TMA)", out, c);
    return 0;
}
