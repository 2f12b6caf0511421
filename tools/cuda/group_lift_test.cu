// group_lift_test.cu — bit-exactness of the 8-lane lifting (lifting_group.cuh)
// against the one-thread register lifting (lifting.cuh) on random lines.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -fmad=false --expt-relaxed-constexpr \
//      -I paper_2302_09883_b200/csrc -I include tools/cuda/group_lift_test.cu -o /tmp/glt
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "lifting_group.cuh"

using namespace wg;

template <int N, int L>
__global__ void k_ref(const double* in, double* fwd, double* inv, int lines) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lines) return;
    double v[N];
    for (int i = 0; i < N; ++i) v[i] = in[l * N + i];
    dwt_line_reg<N, L>(v);
    for (int i = 0; i < N; ++i) fwd[l * N + i] = v[i];
    for (int i = 0; i < N; ++i) v[i] = in[l * N + i];
    idwt_line_reg<N, L>(v);
    for (int i = 0; i < N; ++i) inv[l * N + i] = v[i];
}

template <int N, int L>
__global__ void k_grp(const double* in, double* fwd, double* inv, int lines) {
    constexpr int E = (N - 1) / kGL;
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = gt / kGL, r = gt % kGL;
    const bool ok = l < lines;
    double x[E + 1];
    for (int i = 0; i <= E; ++i) x[i] = ok ? in[l * N + E * r + i] : 0.0;
    dwt_line_grp<N, L>(x, r);
    if (ok)
        for (int i = 0; i <= E; ++i) fwd[l * N + E * r + i] = x[i];
    for (int i = 0; i <= E; ++i) x[i] = ok ? in[l * N + E * r + i] : 0.0;
    idwt_line_grp<N, L>(x, r);
    if (ok)
        for (int i = 0; i <= E; ++i) inv[l * N + E * r + i] = x[i];
}

template <int N, int L>
int run(int lines) {
    std::mt19937_64 rng(N * 100 + L);
    std::uniform_real_distribution<double> U(-2.0, 2.0);
    std::vector<double> h(lines * N);
    for (auto& x : h) x = U(rng);
    for (int k = 0; k < lines; k += 7) h[k * N + (k % N)] = 0.0;  // some exact zeros
    double *in, *f1, *f2, *i1, *i2;
    const size_t b = h.size() * 8;
    cudaMalloc(&in, b); cudaMalloc(&f1, b); cudaMalloc(&f2, b); cudaMalloc(&i1, b); cudaMalloc(&i2, b);
    cudaMemcpy(in, h.data(), b, cudaMemcpyHostToDevice);
    k_ref<N, L><<<(lines + 127) / 128, 128>>>(in, f1, i1, lines);
    k_grp<N, L><<<(lines * kGL + 255) / 256, 256>>>(in, f2, i2, lines);
    std::vector<double> a(h.size()), c(h.size()), d(h.size()), e(h.size());
    cudaMemcpy(a.data(), f1, b, cudaMemcpyDeviceToHost);
    cudaMemcpy(c.data(), f2, b, cudaMemcpyDeviceToHost);
    cudaMemcpy(d.data(), i1, b, cudaMemcpyDeviceToHost);
    cudaMemcpy(e.data(), i2, b, cudaMemcpyDeviceToHost);
    const cudaError_t err = cudaGetLastError();
    const bool ok = err == cudaSuccess && std::memcmp(a.data(), c.data(), b) == 0 && std::memcmp(d.data(), e.data(), b) == 0;
    std::printf("N=%d L=%d %s%s\n", N, L, ok ? "ok" : "MISMATCH", err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaFree(in); cudaFree(f1); cudaFree(f2); cudaFree(i1); cudaFree(i2);
    return ok ? 0 : 1;
}

int main() {
    int bad = 0;
    bad += run<65, 0>(1000); bad += run<65, 1>(1000); bad += run<65, 2>(1000); bad += run<65, 3>(1000);
    bad += run<65, 4>(1000); bad += run<65, 5>(1000); bad += run<65, 6>(1000);
    bad += run<33, 0>(1000); bad += run<33, 2>(1000); bad += run<33, 4>(1000); bad += run<33, 5>(1000);
    bad += run<17, 3>(1000); bad += run<17, 4>(1000);
    std::printf(bad ? "FAILED %d\n" : "ALL OK\n", bad);
    return bad;
}
