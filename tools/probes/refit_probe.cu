// rank_refit_block alone in a one-CTA kernel (224 or 1024 threads), BD_PHASE_TIMING phase prints.
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <numeric>
#include <cuda_runtime.h>
#include "../../paper_2212_02224_b200/csrc/cem_kernels.cuh"
using namespace bd;
__global__ void k(CemState s, const int* order) {
    extern __shared__ __align__(16) unsigned char smem[];
    for (int it = 0; it < 3; ++it) { rank_refit_block(s, 0, order, 0, smem); __syncthreads(); }
}
template <class T> T* dev(const std::vector<T>& h) { T* p; cudaMalloc(&p, h.size() * sizeof(T)); cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice); return p; }
int main(int argc, char** argv) {
    const int B = 1000, d = 8, n = 150, q = 100, T = argc > 1 ? atoi(argv[1]) : 224;
    std::mt19937_64 g(1); std::normal_distribution<double> N01;
    std::vector<double> resid(B), cost(B), params(B * d), xi(B * 22), mean(d, 0.0), cov(d * d, 0.0);
    for (auto& r : resid) r = std::abs(N01(g)); for (auto& c : cost) c = 1000 + 100 * N01(g);
    for (auto& p : params) p = N01(g); for (int i = 0; i < d; ++i) cov[i * d + i] = 1.0;
    std::vector<int> ord(B); std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return resid[a] < resid[b]; });
    CemState s{};
    s.S = 1; s.B = B; s.dim = d; s.n_cons = n; s.n_elite = q; s.iters = 1; s.eta = 0.7; s.gamma = 0.9; s.w_res = 1.0;
    s.mean = dev(mean); s.cov = dev(cov); s.L = dev(cov); s.err = dev(std::vector<int>(1, 0)); s.done = dev(std::vector<int>(1, 0));
    s.resid = dev(resid); s.cost = dev(cost); s.params = dev(params); s.xi = dev(xi);
    s.stats = dev(std::vector<double>(6)); s.best_index = dev(std::vector<long long>(1)); s.best_params = dev(std::vector<double>(d));
    s.best_xi = dev(std::vector<double>(22)); s.best_scal = dev(std::vector<double>(3));
    const int* dord = dev(ord);
    const size_t smem = rank_refit_smem(n, q, d);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<1, T, smem>>>(s, dord);
    printf("rc %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
