// store_micro.cu -- HBM write throughput of the conv-epilogue store patterns:
// a warp owns 32 rows x NCOL fp16 columns of a [rows][C] tensor and writes
// them in column steps of SEG bytes per row (SEG/16 lanes per row, 512/SEG
// rows per STG.128 instruction), vs. a fully contiguous writer.
// build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a tools/store_micro.cu -o tools/store_micro
#include <cstdio>
#include <cstdint>

template <int SEG>
__global__ void rows_kernel(uint4* out, int rows, int C, int tiles_n, int ncol) {
    // block = 8 warps = one 128 x 256 tile (4 row quadrants x 2 column halves), persistent over tiles
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int LPR = SEG / 16, RPI = 32 / LPR;
    const int n_tiles = (rows / 128) * tiles_n;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int m0 = (t / tiles_n) * 128 + (warp & 3) * 32, c0 = (t % tiles_n) * 256 + (warp >> 2) * ncol;
        for (int cb = 0; cb < ncol; cb += SEG / 2) {
#pragma unroll
            for (int k = 0; k < 32 / RPI; ++k) {
                const int r = m0 + k * RPI + lane / LPR;
                const int col = c0 + cb + (lane % LPR) * 8;
                out[(static_cast<int64_t>(r) * C + col) / 8] = make_uint4(r, col, k, cb);
            }
        }
    }
}

__global__ void flat_kernel(uint4* out, int64_t n16) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = make_uint4(i, 0, 1, 2);
}

int main() {
    const int rows = 50176, C = 2048;
    const size_t bytes = size_t(rows) * C * 2;
    uint4* out;
    cudaMalloc(&out, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("%-28s %8.1f us  %6.2f TB/s\n", name, ms * 100, bytes / (ms * 1e-4) / 1e12);
    };
    time("flat (512B per instr)", [&] { flat_kernel<<<148 * 8, 256>>>(out, bytes / 16); });
    time("rows seg 32B (SC=16)", [&] { rows_kernel<32><<<148, 256>>>(out, rows, C, C / 256, 128); });
    time("rows seg 64B (SC=32)", [&] { rows_kernel<64><<<148, 256>>>(out, rows, C, C / 256, 128); });
    time("rows seg 128B", [&] { rows_kernel<128><<<148, 256>>>(out, rows, C, C / 256, 128); });
    time("rows seg 256B", [&] { rows_kernel<256><<<148, 256>>>(out, rows, C, C / 256, 128); });
    time("rows seg 64B x2 CTA/SM", [&] { rows_kernel<64><<<296, 256>>>(out, rows, C, C / 256, 128); });
    time("rows seg 64B x4 CTA/SM", [&] { rows_kernel<64><<<592, 256>>>(out, rows, C, C / 256, 128); });
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
