// norm_micro2.cu -- the norm kernels one at a time inside a CUDA graph (stats
// alone, finalize alone, apply alone), to see where a small layer's time goes.
// build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_1903_05831_b200/csrc \
//        tools/norm_micro2.cu paper_1903_05831_b200/csrc/common.cu -lcuda -o tools/norm_micro2
#include "../paper_1903_05831_b200/csrc/norm.cu"

#include <cstdio>
#include <vector>

using namespace sdb;

#undef CK
#define CK(...)                                                                    \
    do {                                                                           \
        cudaError_t e_ = (__VA_ARGS__);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                          \
        }                                                                          \
    } while (0)

template <class F>
double graph_us(cudaStream_t st, int reps, F&& body) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < reps; ++i) body();
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int w = 0; w < 3; ++w) CK(cudaGraphLaunch(ge, st));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    CK(cudaEventRecord(a, st));
    const int iters = 10;
    for (int w = 0; w < iters; ++w) CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ms * 1e3 / (iters * reps);
}

int main() {
    struct S { long rows; int C; };
    const S shapes[] = {{8400, 256}, {8400, 1024}, {33400, 128}, {133600, 64}, {50176, 2048}};
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::printf("%8s %5s %6s %5s | %8s %8s %8s %8s %8s\n", "rows", "C", "MB", "nblk", "stats", "final", "apply",
                "st+fin", "empty");
    for (const S& s : shapes) {
        const size_t n = static_cast<size_t>(s.rows) * s.C;
        const int L = 20;
        std::vector<void*> x(L), y(L);
        for (int i = 0; i < L; ++i) {
            CK(cudaMalloc(&x[i], n * 2)); CK(cudaMalloc(&y[i], n * 2));
            CK(cudaMemset(x[i], 0x3c, n * 2));
        }
        float *gamma, *beta, *mean, *invstd;
        CK(cudaMalloc(&gamma, s.C * 4)); CK(cudaMalloc(&beta, s.C * 4)); CK(cudaMalloc(&mean, s.C * 4));
        CK(cudaMalloc(&invstd, s.C * 4));
        CK(cudaMemset(gamma, 0, s.C * 4)); CK(cudaMemset(beta, 0, s.C * 4));
        CK(cudaMemset(mean, 0, s.C * 4)); CK(cudaMemset(invstd, 0, s.C * 4));
        void* ws;
        CK(cudaMalloc(&ws, norm_workspace_bytes(s.rows, s.C)));
        const Plan pl = plan_for(s.rows, s.C, 2);
        double* partial = static_cast<double*>(ws);
        int k = 0;
        auto stats = [&] {
            StatArgs sa{};
            sa.a = x[k]; sa.rows = s.rows; sa.C = s.C; sa.partial = partial; sa.slope = 1.f;
            CK(run_stats<__half, 0, 1>(sa, pl, st));
        };
        auto fin = [&] { finalize(partial, pl, s.C, s.rows, 1e-5f, 1, mean, invstd, nullptr, nullptr, nullptr, st); };
        auto apply = [&] {
            ApplyArgs aa{};
            aa.a = x[k]; aa.out = y[k]; aa.gamma = gamma; aa.beta = beta; aa.mean = mean; aa.invstd = invstd;
            aa.slope = 0.01f; aa.act = 2; aa.n8 = n / 8; aa.C = s.C;
            CK(run_apply<__half, 1, 1>(aa, s.rows, pl, st));
        };
        const double t_s = graph_us(st, L, [&] { stats(); k = (k + 1) % L; });
        const double t_f = graph_us(st, L, [&] { fin(); });
        const double t_a = graph_us(st, L, [&] { apply(); k = (k + 1) % L; });
        const double t_sf = graph_us(st, L, [&] { stats(); fin(); k = (k + 1) % L; });
        const double t_e = graph_us(st, L, [&] {
            launch_pdl(finalize_kernel, dim3(1), dim3(32), 0, st, partial, 0, 0, int64_t(1), 1e-5f, 1, mean, invstd,
                       (float*)nullptr, (float*)nullptr, (float*)nullptr);
        });
        std::printf("%8ld %5d %6.1f %5d | %8.2f %8.2f %8.2f %8.2f %8.2f\n", s.rows, s.C, n * 2 / 1e6, pl.nblocks, t_s,
                    t_f, t_a, t_sf, t_e);
        for (int i = 0; i < L; ++i) { cudaFree(x[i]); cudaFree(y[i]); }
        cudaFree(gamma); cudaFree(beta); cudaFree(mean); cudaFree(invstd); cudaFree(ws);
    }
    return 0;
}
