// Pipe-throughput microbenchmark (sm_100a): warp-instructions per cycle per SM for
// FFMA (3-reg), FADD, FMUL, FFMA2, FADD2, mixed FFMA + LOP3, IMAD.  One CTA per SM, 12 warps
// (the fused kernel's occupancy) and 32 warps.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

template <int OP>
__global__ void k(float* out, float a, float b, long long* cyc) {
    float x[CH], y[CH];
    unsigned u[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) { x[i] = threadIdx.x * 1e-3f + i; y[i] = x[i] * 0.5f; u[i] = threadIdx.x + i; }
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (OP == 0) x[i] = __fmaf_rn(x[i], a, y[i]);
            if (OP == 1) x[i] = __fadd_rn(x[i], y[i]);
            if (OP == 2) x[i] = __fmul_rn(x[i], a);
            if (OP == 3) {
                float2 d;
                asm volatile("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
                    "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
                    : "=f"(d.x), "=f"(d.y) : "f"(x[i]), "f"(y[i]), "f"(a), "f"(b), "f"(y[i]), "f"(x[i]));
                x[i] = d.x; y[i] = d.y;
            }
            if (OP == 4) {
                float2 d;
                asm volatile("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
                    "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
                    : "=f"(d.x), "=f"(d.y) : "f"(x[i]), "f"(y[i]), "f"(a), "f"(b));
                x[i] = d.x; y[i] = d.y;
            }
            if (OP == 5) { x[i] = __fmaf_rn(x[i], a, y[i]); u[i] = (u[i] ^ 0x5a5a) + (u[i] >> 3); }
            if (OP == 6) { u[i] = u[i] * 2654435761u + 12345u; }
            if (OP == 7) { u[i] = (u[i] ^ 0x5a5a) + (u[i] >> 3); }
            if (OP == 8) { x[i] = fmaxf(x[i], y[i]) ; y[i] = fminf(y[i], x[i]); }
            if (OP == 9) { x[i] = __shfl_sync(0xffffffffu, x[i], (threadIdx.x + i + 1) & 31); }
            if (OP == 10) { x[i] = __shfl_down_sync(0xffffffffu, x[i], 1); }
            if (OP == 11) { x[i] = (x[i] > y[i]) ? x[i] : y[i] + 1.0f; }
        }
    }
    long long t1 = clock64();
    float s = 0; unsigned us = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) { s += x[i] + y[i]; us += u[i]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)us;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int OP>
void run(const char* name, int nt, double ops_per_inner) {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
    k<OP><<<148, nt>>>(o, 1.0001f, 0.999f, c);
    k<OP><<<148, nt>>>(o, 1.0001f, 0.999f, c);
    cudaDeviceSynchronize();
    long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    double winst = (double)ITERS * CH * ops_per_inner * (nt / 32);
    printf("%-14s warps=%2d  warp-instr/cycle/SM = %.2f  (lane-ops/cycle/SM = %.0f)\n", name, nt / 32, winst / cy,
           winst / cy * 32 * (OP == 3 || OP == 4 ? 2 : 1));
    cudaFree(o); cudaFree(c);
}

int main() {
    for (int nt : {384, 1024}) {
        run<0>("FFMA", nt, 1); run<1>("FADD", nt, 1); run<2>("FMUL", nt, 1); run<3>("FFMA2", nt, 1);
        run<4>("FADD2", nt, 1); run<5>("FFMA+2alu", nt, 3); run<6>("IMAD", nt, 1); run<7>("LOP3/IADD", nt, 2);
        run<8>("FMNMX", nt, 2);
        run<9>("SHFL.IDX", nt, 1);
        run<10>("SHFL.DOWN", nt, 1);
    }
    return 0;
}
