// pipe_bench.cu -- issue/pipe throughput of the instructions K3's softmax and
// epilogue are built from, on one SM: cycles per warp-instruction per SMSP with
// W warps per SMSP, 8 independent dependency chains per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define IT 2048

template <int OP>
__device__ __forceinline__ void op(uint32_t& x, uint32_t c) {
    if (OP == 0) asm volatile("add.s32 %0, %0, %1;" : "+r"(x) : "r"(c));                  // IADD3
    if (OP == 1) asm volatile("mad.lo.s32 %0, %0, %1, %1;" : "+r"(x) : "r"(c));            // IMAD
    if (OP == 2) { float f; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(x)); x = __float_as_uint(f) ^ c; } // I2FP + LOP
    if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(x) : "r"(c));            // FFMA
    if (OP == 4) asm volatile("prmt.b32 %0, %0, %1, 0x3240;" : "+r"(x) : "r"(c));          // PRMT
    if (OP == 5) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(x));                     // MUFU.EX2
    if (OP == 6) asm volatile("max.s32 %0, %0, %1;" : "+r"(x) : "r"(c));                   // IMNMX
    if (OP == 7) asm volatile("max.f32 %0, %0, %1;" : "+r"(x) : "r"(c));                   // FMNMX
    if (OP == 8) asm volatile("lop3.b32 %0, %0, %1, %1, 0x96;" : "+r"(x) : "r"(c));        // LOP3
    if (OP == 9) asm volatile("mul.rn.f32 %0, %0, %1;" : "+r"(x) : "r"(c));                // FMUL
    if (OP == 10) asm volatile("add.rn.f32 %0, %0, %1;" : "+r"(x) : "r"(c));               // FADD
}
template <int OP>
__device__ __forceinline__ void op2(uint64_t& x, uint64_t c) {
    if (OP == 20) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(x) : "l"(c));         // FFMA2
    if (OP == 21) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(c));             // FADD2
    if (OP == 22) asm volatile("fma.rm.f32x2 %0, %0, %1, %1;" : "+l"(x) : "l"(c));         // FFMA2.RM
    if (OP == 23) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(c));             // FMUL2
}

template <int OP>
__global__ void k(uint32_t* out, long long* cyc, uint32_t seed) {
    uint32_t x[CH];
    for (int i = 0; i < CH; ++i) x[i] = seed + threadIdx.x * 7 + i;
    const uint32_t c = seed | 1;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) op<OP>(x[i], c);
    }
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < CH; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}
template <int OP>
__global__ void k2(uint32_t* out, long long* cyc, uint32_t seed) {
    uint64_t x[CH];
    for (int i = 0; i < CH; ++i) x[i] = ((uint64_t)(seed + i) << 32) | (threadIdx.x + i);
    const uint64_t c = 0x3f8000003f800000ull;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) op2<OP>(x[i], c);
    }
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < CH; ++i) s ^= (uint32_t)x[i] ^ (uint32_t)(x[i] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}


// pipe-sharing probes: two instruction kinds interleaved 1:1 on independent chains
template <int M>
__global__ void km(uint32_t* out, long long* cyc, uint32_t seed) {
    uint32_t x[CH], y[CH];
    uint64_t z[CH];
    for (int i = 0; i < CH; ++i) { x[i] = seed + threadIdx.x * 7 + i; y[i] = x[i] * 3; z[i] = ((uint64_t)x[i] << 32) | y[i]; }
    const uint32_t c = seed | 1;
    const uint64_t c2 = 0x3f8000003f800000ull;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (M == 0) { float f; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(x[i])); x[i] = __float_as_uint(f);
                          asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(y[i]) : "r"(c)); }               // I2FP | FFMA
            if (M == 1) { float f; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(x[i])); x[i] = __float_as_uint(f);
                          asm volatile("prmt.b32 %0, %0, %1, 0x3240;" : "+r"(y[i]) : "r"(c)); }              // I2FP | PRMT
            if (M == 2) { asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(z[i]) : "l"(c2));
                          asm volatile("prmt.b32 %0, %0, %1, 0x3240;" : "+r"(y[i]) : "r"(c)); }              // FFMA2 | PRMT
            if (M == 3) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(x[i]));
                          asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(z[i]) : "l"(c2));
                          asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(z[i]) : "l"(c2));
                          asm volatile("prmt.b32 %0, %0, %1, 0x3240;" : "+r"(y[i]) : "r"(c)); }              // MUFU | 2 FFMA2 | PRMT
            if (M == 4) { asm volatile("mad.lo.s32 %0, %0, %1, %1;" : "+r"(x[i]) : "r"(c));
                          asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(y[i]) : "r"(c)); }               // IMAD | FFMA
            if (M == 5) { asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(z[i]) : "l"(c2));
                          asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(y[i]) : "r"(c)); }               // FFMA2 | FFMA
            if (M == 6) { float f; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(x[i])); x[i] = __float_as_uint(f);
                          asm volatile("mad.lo.s32 %0, %0, %1, %1;" : "+r"(y[i]) : "r"(c)); }               // I2FP | IMAD
            if (M == 7) { asm volatile("sub.s32 %0, %0, %1;" : "+r"(x[i]) : "r"(y[i]));
                          asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(y[i]) : "r"(c)); }               // IADD3 | FFMA
            if (M == 8) { asm volatile("sub.s32 %0, %0, %1;" : "+r"(x[i]) : "r"(y[i]));
                          asm volatile("prmt.b32 %0, %0, %1, 0x3240;" : "+r"(y[i]) : "r"(c)); }              // IADD3 | PRMT
            if (M == 9) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(x[i]));
                          float f; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(y[i])); y[i] = __float_as_uint(f) + 1; } // MUFU | I2FP (+IADD)
            if (M == 10) { uint32_t t; asm volatile("sub.s32 %0, %1, %2;" : "=r"(t) : "r"(x[i]), "r"(c)); x[i] = t ^ y[i];
                           asm volatile("sub.s32 %0, %1, %2;" : "=r"(t) : "r"(y[i]), "r"(c)); y[i] = t ^ x[i]; } // 2 x (IADD + LOP)
            if (M == 11) { asm volatile("add.rm.f32x2 %0, %0, %1;" : "+l"(z[i]) : "l"(c2));
                           asm volatile("sub.s32 %0, %0, %1;" : "+r"(x[i]) : "r"(y[i])); }                   // FADD2 | IADD
        }
    }
    long long t1 = clock64();
    uint32_t s = 0;
    for (int i = 0; i < CH; ++i) s ^= x[i] ^ y[i] ^ (uint32_t)z[i] ^ (uint32_t)(z[i] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}

template <typename F>
void run(const char* name, F kern, uint32_t* out, long long* cyc) {
    printf("%-10s", name);
    for (int w : {1, 2, 4}) {
        const int threads = 128 * w; // w warps per SMSP
        kern<<<1, threads>>>(out, cyc, 3u);
        cudaDeviceSynchronize();
        long long h[32];
        cudaMemcpy(h, cyc, sizeof(long long) * threads / 32, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < threads / 32; ++i) mx = h[i] > mx ? h[i] : mx;
        // cycles per warp-instruction per SMSP
        printf("  W=%d %.2f", w, (double)mx / ((double)IT * CH * w));
    }
    printf("\n");
}

int main() {
    uint32_t* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 4096);
    run("IADD3", k<0>, out, cyc);
    run("IMAD", k<1>, out, cyc);
    run("I2FP+LOP", k<2>, out, cyc);
    run("FFMA", k<3>, out, cyc);
    run("PRMT", k<4>, out, cyc);
    run("MUFU.EX2", k<5>, out, cyc);
    run("IMNMX", k<6>, out, cyc);
    run("FMNMX", k<7>, out, cyc);
    run("LOP3", k<8>, out, cyc);
    run("FMUL", k<9>, out, cyc);
    run("FADD", k<10>, out, cyc);
    run("FFMA2", k2<20>, out, cyc);
    run("FADD2", k2<21>, out, cyc);
    run("FFMA2.RM", k2<22>, out, cyc);
    run("FMUL2", k2<23>, out, cyc);
    printf("-- mixes: cycles per (A,B) pair per SMSP\n");
    run("I2FP|FFMA", km<0>, out, cyc);
    run("I2FP|PRMT", km<1>, out, cyc);
    run("FFMA2|PRMT", km<2>, out, cyc);
    run("EX2|2FFMA2|PRMT", km<3>, out, cyc);
    run("IMAD|FFMA", km<4>, out, cyc);
    run("FFMA2|FFMA", km<5>, out, cyc);
    run("I2FP|IMAD", km<6>, out, cyc);
    run("IADD|FFMA", km<7>, out, cyc);
    run("IADD|PRMT", km<8>, out, cyc);
    run("EX2|I2FP+IADD", km<9>, out, cyc);
    run("2x(IADD+LOP)", km<10>, out, cyc);
    run("FADD2|IADD", km<11>, out, cyc);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
