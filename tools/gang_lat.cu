// gang_lat: C-level per-call latency of cdx_gang_priority (no Python) at a few sizes, on the
// persistent path and the multi-launch path.  nvcc ... -o build/gang_lat tools/gang_lat.cu -Lpkg/lib -lcdx
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../include/cdx_c.h"
int main() {
    cdx_ctx* ctx;
    if (cdx_ctx_create(0, &ctx)) return 1;
    const char* only = getenv("GL_N");
    for (uint64_t N : {64ull, 4096ull, 1ull << 20, 1ull << 22}) {
        if (only && strtoull(only, nullptr, 10) != N) continue;
        std::vector<double> arr(N), last(N);
        std::vector<int64_t> sum(N);
        std::vector<uint32_t> cnt(N);
        std::vector<int32_t> knob(N), cap(N);
        std::vector<uint8_t> term(N);
        // config G's distribution (bench.py gang_inputs): exponential gaps (1 ms), service lags
        // ~ Exp(limit/3) so ~5 % escalate, 0-5 iterations of 32-1023 tokens, cap 4-63
        srand(1);
        auto U = [] { return (rand() + 0.5) / (RAND_MAX + 1.0); };
        double t = 0;
        for (uint64_t i = 0; i < N; ++i) {
            t += -1e-3 * std::log(U());
            arr[i] = t;
        }
        const double now_ = t + 1e-3;
        for (uint64_t i = 0; i < N; ++i) {
            last[i] = std::max(0.0, now_ + (0.5 / 3.0) * std::log(U()));
            cnt[i] = rand() % 6; sum[i] = (int64_t)cnt[i] * (32 + rand() % 992);
            cap[i] = 4 + rand() % 60; knob[i] = std::min(cap[i], rand() % 64); term[i] = U() < 0.24;
        }
        t = now_ - 0.1;
        double *da, *dl; int64_t* ds; uint32_t *dc, *order; int32_t *dk, *dp; uint8_t* dt;
        cudaMalloc(&da, N * 8); cudaMalloc(&dl, N * 8); cudaMalloc(&ds, N * 8); cudaMalloc(&dc, N * 4);
        cudaMalloc(&dk, N * 4); cudaMalloc(&dp, N * 4); cudaMalloc(&dt, N); cudaMalloc(&order, N * 4);
        cudaMemcpy(da, arr.data(), N * 8, cudaMemcpyHostToDevice); cudaMemcpy(dl, last.data(), N * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(ds, sum.data(), N * 8, cudaMemcpyHostToDevice); cudaMemcpy(dc, cnt.data(), N * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dk, knob.data(), N * 4, cudaMemcpyHostToDevice); cudaMemcpy(dp, cap.data(), N * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dt, term.data(), N, cudaMemcpyHostToDevice);
        cdx_prog_soa s{da, dl, ds, dc, dk, dp, dt, nullptr, 0, 0};
        cdx_inter_policy pol{};
        pol.order = CDX_ORDER_SJF; pol.starvation_limit = 0.5; pol.prior_tokens = 128.0;
        for (const char* ps : {"1", "0"}) {
            setenv("CDX_GANG_PS", ps, 1);
            uint64_t n = 0;
            for (int w = 0; w < 5; ++w) cdx_gang_priority(ctx, &s, N, &pol, t + 0.1, order, &n, nullptr, nullptr);
            const int reps = N > 100000 ? 50 : 500;
            auto t0 = std::chrono::steady_clock::now();
            for (int r = 0; r < reps; ++r)
                if (cdx_gang_priority(ctx, &s, N, &pol, t + 0.1, order, &n, nullptr, nullptr)) { printf("err %s\n", cdx_last_error(ctx)); return 1; }
            const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps;
            printf("N=%-8llu ps=%s  %.1f us per call (live %llu)\n", (unsigned long long)N, ps, us, (unsigned long long)n);
        }
        cudaFree(da); cudaFree(dl); cudaFree(ds); cudaFree(dc); cudaFree(dk); cudaFree(dp); cudaFree(dt); cudaFree(order);
    }
    return 0;
}
