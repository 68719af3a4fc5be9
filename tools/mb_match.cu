// microbenchmark: warp match / vote throughput on B200 (per SM, cycles per warp-instruction)
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(const uint32_t* in, uint32_t* out, int iters, long long* cyc) {
    uint32_t lane = threadIdx.x & 31;
    uint32_t acc = 0;
    uint32_t v0 = in[(blockIdx.x * blockDim.x + threadIdx.x) & 1023];
    __syncthreads();
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < iters; ++i) {
        #pragma unroll
        for (int j = 0; j < 16; ++j) {
            uint32_t v = v0 + ((i * 16 + j) & 3);  // different per iteration, same per lane pattern
            if (MODE == 0) acc += __match_any_sync(0xffffffffu, v);
            if (MODE == 1) acc += __ballot_sync(0xffffffffu, (v & 1) != 0);
            if (MODE == 2) acc += __match_any_sync(0xffffffffu, v ^ lane);      // all distinct
            if (MODE == 3) acc += __match_any_sync(0xffffffffu, v & 0);         // all equal
            if (MODE == 4) acc += __shfl_sync(0xffffffffu, v, j);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    uint32_t *in, *out; long long* cyc;
    cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 148 * 1024 * 4 * 4); cudaMalloc(&cyc, 148 * 8 * 4);
    uint32_t h[1024]; for (int i = 0; i < 1024; ++i) h[i] = (i * 7) % 5;
    cudaMemcpy(in, h, 4096, cudaMemcpyHostToDevice);
    const char* names[] = {"match(5 distinct)", "ballot", "match(32 distinct)", "match(1 value)", "shfl"};
    for (int mode = 0; mode < 5; ++mode) for (int warps : {8, 16, 32}) {
        int iters = 2000;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        auto launch = [&]() {
            if (mode == 0) k<0><<<148, warps * 32>>>(in, out, iters, cyc);
            if (mode == 1) k<1><<<148, warps * 32>>>(in, out, iters, cyc);
            if (mode == 2) k<2><<<148, warps * 32>>>(in, out, iters, cyc);
            if (mode == 3) k<3><<<148, warps * 32>>>(in, out, iters, cyc);
            if (mode == 4) k<4><<<148, warps * 32>>>(in, out, iters, cyc);
        };
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double ops_per_sm = (double)warps * iters * 16;
        printf("%-20s warps/SM=%2d  %.3f ms  %.2f cycles per warp-op per SM (clock64 %.2f)\n", names[mode], warps, ms,
               ms * 1e-3 * 1.965e9 / ops_per_sm, (double)c / ops_per_sm);
    }
    return 0;
}
