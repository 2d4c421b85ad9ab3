// conv_micro.cu -- one conv shape through the C++ entry points, timed inside a
// CUDA graph: fprop, plain dgrad, dgrad + residual addend + activation mask, wgrad.
// usage: conv_micro N H W C K R S stride pad [reps]
// build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_1903_05831_b200/csrc \
//        tools/conv_micro.cu -L paper_1903_05831_b200 -lsdb -lcuda -o tools/conv_micro
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sdb_internal.h"

#define CK(...)                                                                    \
    do {                                                                           \
        cudaError_t e_ = (__VA_ARGS__);                                            \
        if (e_ != cudaSuccess) {                                                   \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                          \
        }                                                                          \
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
    CK(cudaGraphLaunch(ge, st));
    CK(cudaStreamSynchronize(st));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    CK(cudaEventRecord(a, st));
    const int iters = 5;
    for (int w = 0; w < iters; ++w) CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ms * 1e3 / (iters * reps);
}

int main(int argc, char** argv) {
    if (argc < 10) {
        std::printf("usage: conv_micro N H W C K R S stride pad [reps] [which: a=all f d m w]\n");
        return 2;
    }
    sdb::ConvShape g{};
    g.N = std::atoi(argv[1]); g.H = std::atoi(argv[2]); g.W = std::atoi(argv[3]); g.C = std::atoi(argv[4]);
    g.K = std::atoi(argv[5]); g.R = std::atoi(argv[6]); g.S = std::atoi(argv[7]);
    g.stride = std::atoi(argv[8]); g.pad = std::atoi(argv[9]);
    const int reps = argc > 10 ? std::atoi(argv[10]) : 10;
    const char* which = argc > 11 ? argv[11] : "fdmw";
    const size_t nx = size_t(g.N) * g.H * g.W * g.C, ny = size_t(g.N) * g.Ho() * g.Wo() * g.K,
                 nw = size_t(g.K) * g.R * g.S * g.C;
    void *x, *y, *w, *dx, *mask, *add, *dw, *ws, *mbits;
    CK(cudaMalloc(&mbits, nx / 8 + 16)); CK(cudaMemset(mbits, 0xa5, nx / 8 + 16));
    CK(cudaMalloc(&x, nx * 2)); CK(cudaMalloc(&dx, nx * 2)); CK(cudaMalloc(&mask, nx * 2)); CK(cudaMalloc(&add, nx * 2));
    CK(cudaMalloc(&y, ny * 2)); CK(cudaMalloc(&w, nw * 2)); CK(cudaMalloc(&dw, nw * 2));
    const size_t wsb = sdb::conv_wgrad_workspace(g, 1) + 256;
    CK(cudaMalloc(&ws, wsb));
    CK(cudaMemset(x, 0x1c, nx * 2)); CK(cudaMemset(mask, 0x3c, nx * 2)); CK(cudaMemset(add, 0x1c, nx * 2));
    CK(cudaMemset(y, 0x1c, ny * 2)); CK(cudaMemset(w, 0x1c, nw * 2));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    const double fl = 2.0 * g.N * g.Ho() * g.Wo() * double(g.K) * g.C * g.R * g.S;
    auto rep = [&](const char* name, double us, double bytes) {
        std::printf("%-10s %9.2f us  %7.1f TF/s  %7.1f GB/s (algorithmic)\n", name, us, fl / us / 1e6, bytes / us / 1e3);
    };
    for (const char* p = which; *p; ++p) {
        if (*p == 'f')
            rep("fprop", graph_us(st, reps, [&] { CK(sdb::conv_fprop(g, 1, x, w, y, st)); }), 2.0 * (nx + ny + nw));
        if (*p == 'd')
            rep("dgrad", graph_us(st, reps, [&] { CK(sdb::conv_dgrad(g, 1, y, w, dx, 0, st)); }), 2.0 * (nx + ny + nw));
        if (*p == 'm')
            rep("dgrad+a+m", graph_us(st, reps, [&] { CK(sdb::conv_dgrad(g, 1, y, w, dx, 1, st, add, mask, 0.01f)); }),
                2.0 * (3 * nx + ny + nw));
        if (*p == 'b')
            rep("dgrad+a+bits", graph_us(st, reps, [&] {
                    CK(sdb::conv_dgrad(g, 1, y, w, dx, 1, st, add, mask, 0.01f, static_cast<const uint8_t*>(mbits)));
                }),
                2.0 * (2 * nx + ny + nw) + nx / 8.0);
        if (*p == 'w')
            rep("wgrad", graph_us(st, reps, [&] { CK(sdb::conv_wgrad(g, 1, x, y, dw, ws, wsb, st)); }),
                2.0 * (nx + ny + nw));
    }
    return 0;
}
