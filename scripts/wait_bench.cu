// wait_bench.cu -- cost of mbarrier waiting flavours on a B200 SMSP: while one
// warp waits (~200 us) on an mbarrier, 1 or 2 compute warps on the SAME SMSP run
// a fixed FFMA loop; reports the compute slowdown vs no waiter, the waiter's
// loop iterations, and the wake-up latency after the arrive.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wait_bench wait_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ bool try_wait_hint(uint32_t bar, uint32_t par, uint32_t ns) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(par), "r"(ns) : "memory");
    return ok;
}
__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0, 1, 0, P;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// warps: 0 = waiter (lane 0 waits, mode), 4 = arriver (SMSP 0; sleeps then arrives), compute warps 8, 12 (SMSP 0)
__global__ void k(int mode, int ncomp, long long* out, int iters) {
    __shared__ __align__(8) uint64_t mb;
    __shared__ unsigned long long t_arrive;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&mb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (warp == 0) {
        if (mode == 0) return; // no waiter
        long long n = 0;
        if (lane == 0) {
            if (mode == 1) { while (!try_wait(bar, 0)) ++n; }
            else if (mode == 2) { while (!try_wait_hint(bar, 0, 1000000)) ++n; }
            else if (mode == 3) { while (!try_wait(bar, 0)) { __nanosleep(512); ++n; } }
            else if (mode == 4) { while (!try_wait(bar, 0)) { __nanosleep(2000); ++n; } }
            else if (mode == 5) { while (!test_wait(bar, 0)) ++n; }
            else if (mode == 6) { while (!try_wait_hint(bar, 0, 0x989680)) ++n; }
            const uint64_t t1 = gtime();
            out[0] = n;
            out[1] = (long long)(t1 - t_arrive);
        }
        __syncwarp();
    } else if (warp == 4) {
        if (lane == 0) {
            const uint64_t t0 = gtime();
            while (gtime() - t0 < 200000) __nanosleep(1000);
            t_arrive = gtime();
            __threadfence_block();
            asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(bar) : "memory");
        }
    } else if ((warp == 8 && ncomp >= 1) || (warp == 12 && ncomp >= 2)) {
        float a = lane, b = 1.0001f, c = 0.5f, d = lane * 2, e = 3, f = 4, g = 5, h = 6;
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            a = fmaf(a, b, c); d = fmaf(d, b, c); e = fmaf(e, b, c); f = fmaf(f, b, c);
            g = fmaf(g, b, c); h = fmaf(h, b, c);
        }
        const long long t1 = clock64();
        if (lane == 0) out[2 + (warp == 12)] = t1 - t0;
        if (a + d + e + f + g + h == 0.123f) out[5] = 1;
    }
}

int main() {
    long long* d; cudaMalloc(&d, 64);
    const char* names[] = {"none", "try_wait spin", "try_wait hint 1ms", "try_wait+nanosleep512", "try_wait+nanosleep2000", "test_wait spin", "try_wait hint 10M"};
    for (int nc = 1; nc <= 2; ++nc)
    for (int m = 0; m < 7; ++m) {
        cudaMemset(d, 0, 64);
        k<<<1, 512>>>(m, nc, d, 50000);
        cudaDeviceSynchronize();
        long long h[6]; cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
        printf("compute warps %d  %-24s waiter iters %8lld  wake latency %6lld ns  compute cycles %lld %lld\n", nc, names[m], h[0], h[1], h[2], h[3]);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
