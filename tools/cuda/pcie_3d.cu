// pcie_3d.cu — host<->device copy throughput of a patch grid buffer: whole
// (N+2)^2 blocks contiguous vs only the logical N x N cells (3-D copy with
// pitches), pinned host memory.  nvcc -O3 -o pcie_3d pcie_3d.cu
#include <cstdio>
#include <cuda_runtime.h>

int main() {
    const size_t N = 65, TP = N + 2, blocks = 9 * 4096;  // 36864 blocks = 1.32 GB of grid buffer
    const size_t bytes = blocks * TP * TP * 8;
    double *h, *d;
    cudaMallocHost(&h, bytes);
    cudaMalloc(&d, bytes);
    for (size_t i = 0; i < bytes / 8; i += 4096) h[i] = 1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto rate = [&](const char* name, auto&& f, double moved) {
        f();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int k = 0; k < 3; ++k) f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s %8.2f GB/s (%s)\n", name, 3 * moved / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    rate("H2D contiguous", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice); }, bytes);
    rate("D2H contiguous", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); }, bytes);
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(h + TP + 1, TP * 8, N * 8, TP);
    p.dstPtr = make_cudaPitchedPtr(d + TP + 1, TP * 8, N * 8, TP);
    p.extent = make_cudaExtent(N * 8, N, blocks);
    p.kind = cudaMemcpyHostToDevice;
    const double logical = (double)blocks * N * N * 8;
    rate("H2D logical (3-D)", [&] { cudaMemcpy3DAsync(&p); }, logical);
    cudaMemcpy3DParms q = p;
    q.srcPtr = p.dstPtr;
    q.dstPtr = p.srcPtr;
    q.kind = cudaMemcpyDeviceToHost;
    rate("D2H logical (3-D)", [&] { cudaMemcpy3DAsync(&q); }, logical);
    printf("logical / whole bytes = %.4f\n", logical / bytes);
    return 0;
}
