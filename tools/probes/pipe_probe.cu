// Issue-rate probes for the K5 redesign: FFMA (register operands) vs FFMA2 (packed f32x2)
// vs FFMA + ALU mix, in warp-instructions per clock per SM.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 pipe_probe.cu -o pipe_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int U = 16;

__global__ void k_ffma(float* out, const float* in, int iters) {
    float a = in[0], b = in[1];
    float x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma2(float* out, const float* in, int iters) {
    float2 a = make_float2(in[0], in[2]), b = make_float2(in[1], in[3]);
    float2 x[8];
    for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x + k, threadIdx.x - k);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], a, b);
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
    if (s == 1234.5f) out[0] = s;
}

__global__ void k_mix(float* out, const float* in, int iters) {
    float a = in[0], b = in[1];
    float x[8];
    unsigned y[8];
    for (int k = 0; k < 8; ++k) {
        x[k] = threadIdx.x + k;
        y[k] = threadIdx.x * 7 + k;
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                x[k] = fmaf(x[k], a, b);
                y[k] = (y[k] ^ 0x5bd1e995u) & (y[k] >> 1 | 0x10u);
            }
    float s = 0;
    unsigned t = 0;
    for (int k = 0; k < 8; ++k) {
        s += x[k];
        t ^= y[k];
    }
    if (s == 1234.5f || t == 77u) out[0] = s + t;
}

__global__ void k_fsetp(float* out, const float* in, int iters) {
    float a = in[0], b = in[1];
    float x[8];
    int c = 0;
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                x[k] = fmaf(x[k], a, b);
                c += (x[k] > b) ? 1 : 0;
            }
    float s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5f || c == 77) out[0] = s + c;
}

template <typename K>
void run(const char* name, K k, double ops_per_inner, float* out, const float* in) {
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<blocks, threads>>>(out, in, 64);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k<<<blocks, threads>>>(out, in, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double warps = (double)blocks * threads / 32;
    const double winst = warps * iters * U * ops_per_inner;  // warp-instructions of the loop body
    const double cycles = best * 1e-3 * clk * 1e3;
    printf("%-8s %.3f ms  %.3f warp-instr/clk/SM  (%d kHz)\n", name, best, winst / cycles / 148.0, clk);
}

int main() {
    float *out, *in;
    cudaMalloc(&out, 64);
    cudaMalloc(&in, 64);
    float h[4] = {0.999999f, 1e-6f, 0.999998f, 2e-6f};
    cudaMemcpy(in, h, 16, cudaMemcpyHostToDevice);
    run("ffma", k_ffma, 8, out, in);
    run("ffma2", k_ffma2, 8, out, in);
    run("mix", k_mix, 8 * 4, out, in);  // ffma + (lop3/shf/...) ~3 ALU
    run("fsetp", k_fsetp, 8 * 3, out, in);
    return 0;
}
