// stem_micro.cu -- the stem's im2col staging kernel alone, timed in a CUDA graph
// build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_1903_05831_b200/csrc \
//        tools/stem_micro.cu -L paper_1903_05831_b200 -lsdb -o tools/stem_micro
#include <cstdio>
#include <cstdlib>

#include "detect.h"

int main() {
    const int N = 2, H = 800, W = 1333, Ho = 400, Wo = 667;
    void *x, *out;
    cudaMalloc(&x, size_t(N) * H * W * 8 * 2);
    cudaMalloc(&out, size_t(N) * Ho * Wo * 192 * 2);
    cudaMemset(x, 0x1c, size_t(N) * H * W * 8 * 2);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    sdb::stem_im2col(x, N, H, W, 8, Ho, Wo, 2, 3, out, st);
    cudaStreamSynchronize(st);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 10; ++i) sdb::stem_im2col(x, N, H, W, 8, Ho, Wo, 2, 3, out, st);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / 50;
    std::printf("stem_im2col %.2f us  (%.2f TB/s of X' writes)  %s\n", us, N * Ho * Wo * 384.0 / us / 1e6,
                cudaGetErrorString(cudaGetLastError()));
    return 0;
}
