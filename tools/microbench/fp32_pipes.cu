// FP32 pipe throughput on sm_100a by operand form: how many warp
// instructions per cycle per SM sub-partition (SMSP) FFMA / FFMA2 / FMUL2 /
// FADD2 issue when their operands are registers, constant-bank operands, or
// the same register pair reused.  Guides the bump-body encoding of the march
// kernels (rr_march.cuh accel_bumps_x2).  8 independent chains per thread,
// 148 x 8 CTAs x 256 threads, clock64() cycles of the timed loop.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp32p fp32_pipes.cu && /tmp/fp32p
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }

struct Args { float a, b; u64 a2, b2; };
static u64 pk_host(float a, float b) {
    u64 r;
    unsigned ua, ub;
    memcpy(&ua, &a, 4);
    memcpy(&ub, &b, 4);
    r = (u64)ua | ((u64)ub << 32);
    return r;
}

constexpr int CH = 8, REP = 16;

template <int OP>
__global__ void __launch_bounds__(256) pipe_kernel(const __grid_constant__ Args A, int iters, float* sink,
                                                   long long* cycles, const float* in) {
    float x[CH], y[CH], z[CH];
    u64 X[CH], Y[CH], Z[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        // run-time values (from memory), so no operand folds into an immediate
        x[i] = in[(threadIdx.x + 3 * i) & 63];
        y[i] = in[64 + ((threadIdx.x + i) & 63)];
        z[i] = in[128 + ((threadIdx.x + 5 * i) & 63)];
        X[i] = pk(x[i], x[i] + 0.5f);
        Y[i] = pk(y[i], y[i] * 0.999f);
        Z[i] = pk(z[i], z[i] * 2.f);
    }
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < REP; ++r) {
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                if (OP == 0) x[i] = ffma(x[i], y[i], z[i]);          // FFMA R,R,R
                if (OP == 1) x[i] = ffma(x[i], A.a, z[i]);           // FFMA R,c,R
                if (OP == 2) x[i] = ffma(x[i], A.a, A.b);            // FFMA R,c,c (probe form)
                if (OP == 3) X[i] = fma2(X[i], Y[i], Z[i]);          // FFMA2 R,R,R
                if (OP == 4) X[i] = fma2(X[i], A.a2, Z[i]);          // FFMA2 R,c,R
                if (OP == 5) X[i] = fma2(X[i], A.a2, A.b2);          // FFMA2 R,c,c
                if (OP == 6) X[i] = mul2(X[i], Y[i]);                // FMUL2 R,R
                if (OP == 7) X[i] = add2(X[i], Z[i]);                // FADD2 R,R
                if (OP == 8) X[i] = fma2(X[i], X[i], Z[i]);          // FFMA2 R,R(same),R
                if (OP == 9) X[i] = mul2(X[i], A.a2);                // FMUL2 R,c
                if (OP == 10) X[i] = fma2(X[i], pk(y[i], y[i]), Z[i]); // FFMA2 R,R.F32(bcast),R
                if (OP == 11) X[i] = fma2(X[i], pk(A.a, A.a), Z[i]);   // FFMA2 R,UR.F32(bcast),R
                if (OP == 12) X[i] = fma2(X[i], (i & 1) ? pk(A.b, A.b) : pk(A.a, A.a), Z[i]);  // both halves of one UR pair
                if (OP == 13) X[i] = add2(X[i], pk(A.a, A.a));         // FADD2 R,UR.F32(bcast)
            }
        }
    }
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        float a, b;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(X[i]));
        s += x[i] + a + b;
    }
    if (s == 12345.678f) sink[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = t1 - t0;
}

template <int OP>
void run(const char* name, int lanes_per_inst) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* sink;
    long long* cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, 8);
    float hin[192];
    for (int k = 0; k < 64; ++k) {
        hin[k] = 0.001f * k;
        hin[64 + k] = 1.0000001f + 1e-8f * k;
        hin[128 + k] = 1e-7f * (k + 1);
    }
    float* din;
    cudaMalloc(&din, sizeof hin);
    cudaMemcpy(din, hin, sizeof hin, cudaMemcpyHostToDevice);
    Args A{1.0000001f, 1e-7f, pk_host(1.0000001f, 1.0000002f), pk_host(1e-7f, 2e-7f)};
    const int blocks = sms * 8, iters = 2048;
    pipe_kernel<OP><<<blocks, 256>>>(A, 16, sink, cyc, din);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    pipe_kernel<OP><<<blocks, 256>>>(A, iters, sink, cyc, din);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double warp_inst = (double)CH * REP * iters * blocks * 256 / 32;
    const double per_smsp_s = warp_inst / (sms * 4) / (ms * 1e-3);
    // warp instructions per cycle per SMSP, from block 0's clock64 span (its
    // SM runs 8 CTAs = 64 warps = 16 per SMSP for the whole span)
    const double inst_per_cyc = (double)CH * REP * iters * 16 / (double)c;
    printf("%-22s %7.3f ms  %6.3f warp-inst/clk/SMSP (clock64)  %8.1f G warp-inst/s/SMSP  %6.2f TFLOP/s(lanes x2)\n",
           name, ms, inst_per_cyc, per_smsp_s / 1e9, warp_inst * 32 * lanes_per_inst * 2 / (ms * 1e-3) / 1e12);
    cudaFree(sink);
    cudaFree(cyc);
    cudaFree(din);
}

int main() {
    run<0>("FFMA  R,R,R", 1);
    run<1>("FFMA  R,c,R", 1);
    run<2>("FFMA  R,c,c", 1);
    run<3>("FFMA2 R,R,R", 2);
    run<4>("FFMA2 R,c,R", 2);
    run<5>("FFMA2 R,c,c", 2);
    run<6>("FMUL2 R,R", 2);
    run<7>("FADD2 R,R", 2);
    run<8>("FFMA2 R,R(same),R", 2);
    run<9>("FMUL2 R,c", 2);
    run<10>("FFMA2 R,Rbcast,R", 2);
    run<11>("FFMA2 R,URbcast,R", 2);
    run<12>("FFMA2 R,URbcast2,R", 2);
    run<13>("FADD2 R,URbcast", 2);
    return 0;
}
