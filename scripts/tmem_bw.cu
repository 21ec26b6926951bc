// tmem_bw.cu -- TMEM load / store throughput on one SM: W warps (W/4 per lane
// quadrant) each issue R rounds of tcgen05.ld (or .st) 32x32b.x32 (4 KB per warp
// instruction) with a wait per round; reports bytes per SM clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                 "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                 "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                 "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}

__global__ void k(int mode, int rounds, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t tptr;
    const int warp = threadIdx.x >> 5;
    if (warp == 0)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tptr)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tptr + (((warp & 3) * 32) << 16) + ((warp >> 2) & 7) * 64;
    uint32_t r[32], acc = 0;
    for (int i = 0; i < 32; ++i) r[i] = threadIdx.x + i;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < rounds; ++it) {
        if (mode == 0) {
            ld32(tm, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += r[0] ^ r[31];
        } else if (mode == 1) {
            st32(tm, r);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        } else { // two loads per wait
            uint32_t r2[32];
            ld32(tm, r);
            ld32(tm + 32, r2);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc += r[0] ^ r2[31];
        }
    }
    long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tptr));
}

int main() {
    unsigned long long* d; uint32_t* s; cudaMalloc(&d, 8 * 1024); cudaMalloc(&s, 4 << 20);
    const int rounds = 4096;
    for (int mode = 0; mode < 3; ++mode)
        for (int w : {4, 8, 16}) {
            k<<<148, 32 * w>>>(mode, rounds, d, s);
            cudaDeviceSynchronize();
            unsigned long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
            const double bytes = (double)w * rounds * 4096.0 * (mode == 2 ? 2 : 1);
            printf("%s warps %2d: %.1f B/clk per SM (%.0f cycles per warp-instr round)\n",
                   mode == 0 ? "ld x32  " : (mode == 1 ? "st x32  " : "ld 2xx32"), w, bytes / cyc, cyc / rounds);
        }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
