// norm_micro.cu -- per-layer cost of the norm passes inside a CUDA graph (the
// way the training step runs them), for the R50-C4 layer shapes.
// build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_1903_05831_b200/csrc \
//        tools/norm_micro.cu -L paper_1903_05831_b200 -lsdb -Xlinker -rpath=paper_1903_05831_b200 -o tools/norm_micro
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sdb_internal.h"

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)

template <class F>
double graph_us(cudaStream_t st, int reps, F&& body) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    body();  // eager first call (lazy per-device scratch is allocated outside the capture)
    CK(cudaStreamSynchronize(st));
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
    const S shapes[] = {{8400, 256}, {8400, 1024}, {33400, 128}, {33400, 512}, {133600, 64}, {133600, 256},
                        {50176, 512}, {50176, 2048}};
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::printf("%8s %5s %8s | %9s %9s %9s %9s | us per layer (graph of 20 layers, distinct buffers)\n", "rows", "C",
                "MB", "fwd", "stats", "bwd", "apply_add");
    for (const S& s : shapes) {
        const size_t n = static_cast<size_t>(s.rows) * s.C;
        const int L = 20;
        std::vector<void*> x(L), y(L), dy(L), dx(L), o2(L);
        for (int i = 0; i < L; ++i) {
            CK(cudaMalloc(&x[i], n * 2)); CK(cudaMalloc(&y[i], n * 2)); CK(cudaMalloc(&dy[i], n * 2));
            CK(cudaMalloc(&dx[i], n * 2)); CK(cudaMalloc(&o2[i], n * 2));
            CK(cudaMemset(x[i], 0x3c, n * 2)); CK(cudaMemset(y[i], 0x3c, n * 2)); CK(cudaMemset(dy[i], 0x3c, n * 2));
        }
        float *gamma, *beta, *mean, *invstd, *dg, *db;
        CK(cudaMalloc(&gamma, s.C * 4)); CK(cudaMalloc(&beta, s.C * 4)); CK(cudaMalloc(&mean, s.C * 4));
        CK(cudaMalloc(&invstd, s.C * 4)); CK(cudaMalloc(&dg, s.C * 4)); CK(cudaMalloc(&db, s.C * 4));
        std::vector<float> one(s.C, 1.0f);
        CK(cudaMemcpy(gamma, one.data(), s.C * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(invstd, one.data(), s.C * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(beta, 0, s.C * 4)); CK(cudaMemset(mean, 0, s.C * 4));
        void* ws;
        CK(cudaMalloc(&ws, sdb::norm_workspace_bytes(s.rows, s.C)));
        int k = 0;
        const double f = graph_us(st, L, [&] {
            CK(sdb::bn_forward(1, x[k], gamma, beta, y[k], mean, invstd, s.rows, s.C, 1e-5f, 2, 0.01f, ws, st));
            k = (k + 1) % L;
        });
        const double t = graph_us(st, L, [&] {
            CK(sdb::bn_forward_stats(1, x[k], mean, invstd, s.rows, s.C, 1e-5f, 2, ws, st));
            k = (k + 1) % L;
        });
        const double b = graph_us(st, L, [&] {
            CK(sdb::iabn_backward(1, dy[k], y[k], gamma, beta, mean, invstd, dx[k], dg, db, s.rows, s.C, 0.01f, ws,
                                  st));
            k = (k + 1) % L;
        });
        const double a = graph_us(st, L, [&] {
            CK(sdb::bn_apply_add_act(1, x[k], gamma, beta, mean, invstd, y[k], dy[k], o2[k], s.rows, s.C, 0.01f, 2,
                                     0.01f, st));
            k = (k + 1) % L;
        });
        std::printf("%8ld %5d %8.1f | %9.2f %9.2f %9.2f %9.2f   (fwd %5.0f GB/s, bwd %5.0f GB/s)\n", s.rows, s.C,
                    n * 2 / 1e6, f, t, b, a, 3.0 * n * 2 / (f * 1e3), 5.0 * n * 2 / (b * 1e3));
        for (int i = 0; i < L; ++i) { cudaFree(x[i]); cudaFree(y[i]); cudaFree(dy[i]); cudaFree(dx[i]); cudaFree(o2[i]); }
        cudaFree(gamma); cudaFree(beta); cudaFree(mean); cudaFree(invstd); cudaFree(dg); cudaFree(db); cudaFree(ws);
    }
    return 0;
}
