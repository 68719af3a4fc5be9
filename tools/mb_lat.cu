// latency microbenchmark: dependent chains of MATCH.ANY / VOTE / LDS / DADD (1 warp)
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* io, double* dio, long long* out, int n) {
    __shared__ uint32_t sm[1024];
    uint32_t lane = threadIdx.x;
    sm[lane] = lane & 3;
    __syncwarp();
    uint32_t v = io[lane];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) v = __match_any_sync(0xffffffffu, v) & 3;
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) v = __ballot_sync(0xffffffffu, v & 1) & 3;
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) v = sm[v & 31];
    long long t3 = clock64();
    double d = dio[lane];
    for (int i = 0; i < n; ++i) d = __dsub_rn(d, 1e-30);
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) d = __ddiv_rn(d, 1.0000001);
    long long t5 = clock64();
    io[lane] = v; dio[lane] = d;
    if (lane == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; }
}
int main() {
    uint32_t* io; double* dio; long long* out;
    cudaMalloc(&io, 128); cudaMalloc(&dio, 256); cudaMalloc(&out, 64);
    cudaMemset(io, 0, 128); cudaMemset(dio, 0, 256);
    int n = 1000;
    k<<<1, 32>>>(io, dio, out, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(io, dio, out, n); cudaDeviceSynchronize();
    long long h[5]; cudaMemcpy(h, out, 40, cudaMemcpyDeviceToHost);
    const char* nm[] = {"MATCH.ANY", "VOTE(ballot)", "LDS", "DADD", "DDIV"};
    for (int i = 0; i < 5; ++i) printf("%-14s latency ~ %.1f cycles\n", nm[i], (double)h[i] / n);
}
