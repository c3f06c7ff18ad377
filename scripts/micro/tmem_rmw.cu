// Microbenchmark: fp64 read-modify-write throughput of a per-pixel class accumulator held in
// shared memory (LDS.128/STS.128, 2 px per lane) vs tensor memory (tcgen05.ld/st 32x32b.x2,
// 1 px per lane), and both at once. Decides whether TMEM can take part of the raster's
// semantic scatter. Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int C = 102;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int MODE, int B>
__global__ void __launch_bounds__(256) k(int iters, double* out, unsigned long long* cyc) {
    extern __shared__ double2 acc[];  // [C][32]
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < C * 32; i += blockDim.x) acc[i] = make_double2(0.0, 0.0);
    if (MODE != 0) {
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" :: "r"(smem_u32(&tbase)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    } else {
        __syncthreads();
    }
    const uint32_t tb = (MODE != 0) ? tbase + ((32u * (warp & 3)) << 16) : 0u;
    // zero the TMEM columns this warp uses
    if (MODE != 0) {
        for (int c = 0; c < 256; c += 2) {
            uint32_t z = 0;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" :: "r"(tb + c), "r"(z), "r"(z));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    const double w0 = 1e-3 * (lane + 1), w1 = 2e-3 * (lane + 1);
    unsigned long long t0 = clock64();
    uint32_t cls = warp * 13;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0 || MODE == 2) {  // smem: B classes, 2 px per lane
#pragma unroll
            for (int j = 0; j < B; ++j) {
                const uint32_t c = (cls + 37u * j) % C;
                double2 a = acc[c * 32 + lane];
                a.x += w0;
                a.y += w1;
                acc[c * 32 + lane] = a;
            }
        }
        if (MODE == 1 || MODE == 2) {  // tmem: B classes, 1 px per lane (fp64 = 2 columns)
            uint32_t r[2 * B];
#pragma unroll
            for (int j = 0; j < B; ++j) {
                const uint32_t c = (cls + 41u * j + 5u) % 96u;  // 96 fp64 columns pairs in 256 cols? use < 128
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n"
                             : "=r"(r[2 * j]), "=r"(r[2 * j + 1]) : "r"(tb + 2 * c));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
            for (int j = 0; j < B; ++j) {
                double v = __hiloint2double(r[2 * j + 1], r[2 * j]);
                v += w0;
                r[2 * j] = __double2loint(v);
                r[2 * j + 1] = __double2hiint(v);
            }
#pragma unroll
            for (int j = 0; j < B; ++j) {
                const uint32_t c = (cls + 41u * j + 5u) % 96u;
                asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n"
                             :: "r"(tb + 2 * c), "r"(r[2 * j]), "r"(r[2 * j + 1]));
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
        cls = (cls * 1103515245u + 12345u) >> 8;
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    double s = 0.0;
    if (MODE != 1)
        for (int i = threadIdx.x; i < C * 32; i += blockDim.x) s += acc[i].x + acc[i].y;
    if (MODE != 0) {
        uint32_t a, b;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(a), "=r"(b) : "r"(tb + 10));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        s += __hiloint2double(b, a);
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" :: "r"(tbase));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int B>
void run(const char* name, int ctas_per_sm) {
    const int sms = 148, grid = sms * ctas_per_sm, iters = 4000;
    double* out;
    unsigned long long* cyc;
    cudaMalloc(&out, sizeof(double) * grid * 256);
    cudaMalloc(&cyc, sizeof(unsigned long long) * grid);
    const int smem = C * 32 * 16;
    cudaFuncSetAttribute(k<MODE, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<MODE, B><<<grid, 256, smem>>>(10, out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE, B><<<grid, 256, smem>>>(iters, out, cyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h = 0;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    // pixel-updates: smem B x 64 px per warp per iter; tmem B x 32 px per warp per iter
    double upd = 0;
    if (MODE == 0 || MODE == 2) upd += double(grid) * 8 * iters * B * 64;
    if (MODE == 1 || MODE == 2) upd += double(grid) * 8 * iters * B * 32;
    const double per_sm_cycle = upd / (ms * 1e-3) / sms / 1.965e9;
    printf("%-28s ctas/sm=%d B=%2d  %8.3f ms  %6.2f px-updates/SM/cycle (clk/CTA %llu)  err=%s\n", name,
           ctas_per_sm, B, ms, per_sm_cycle, h, cudaGetErrorString(err));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int cps : {1, 2}) {
        run<0, 8>("smem LDS/STS.128", cps);
        run<1, 8>("tmem ld/st.x2", cps);
        run<1, 16>("tmem ld/st.x2", cps);
        run<2, 8>("smem + tmem", cps);
    }
    return 0;
}
