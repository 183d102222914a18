// Write-pattern microbenchmark: 12 GB of int4 stores laid out as the lattice
// fill writes them. (a) grid-stride linear; (b) warp chunks of CH bytes written sequentially,
// chunks assigned grid-stride; (c) block chunks of CH bytes.  nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a write_pattern.cu -o wp && ./wp
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_linear(int4 *p, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_int4((int)i, 1, 2, 3);
}
__global__ void k_warpchunk(int4 *p, size_t n16, size_t ch16) {
    const int lane = threadIdx.x & 31;
    const size_t nch = n16 / ch16;
    const size_t w0 = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, ws = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t c = w0; c < nch; c += ws)
        for (size_t i = lane; i < ch16; i += 32) p[c * ch16 + i] = make_int4((int)i, 1, 2, 3);
}
__global__ void k_blockchunk(int4 *p, size_t n16, size_t ch16) {
    const size_t nch = n16 / ch16;
    for (size_t c = blockIdx.x; c < nch; c += gridDim.x)
        for (size_t i = threadIdx.x; i < ch16; i += blockDim.x) p[c * ch16 + i] = make_int4((int)i, 1, 2, 3);
}
// two arrays written together, as the lattice fill does: per 128-entry group, one int4 per lane
// into A (4 B/entry) and two 16-byte stores per lane into B (8 B/entry), chunks of ch entries
__global__ void k_two(int4 *A, int4 *B, size_t nent, size_t ch) {
    const int lane = threadIdx.x & 31;
    const size_t nch = nent / ch;
    const size_t w0 = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, ws = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t c = w0; c < nch; c += ws)
        for (size_t g = 0; g < ch; g += 128) {
            const size_t e = c * ch + g;
            A[(e >> 2) + lane] = make_int4((int)e, 1, 2, 3);
            B[(e >> 1) + lane] = make_int4((int)e, 4, 5, 6);
            B[(e >> 1) + 32 + lane] = make_int4((int)e, 7, 8, 9);
        }
}
int main() {
    const size_t bytes = 12ull << 30, n16 = bytes / 16;
    int4 *p;
    cudaMalloc(&p, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char *name, auto fn) {
        fn();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("{\"pattern\": \"%s\", \"ms\": %.3f, \"gbs\": %.1f}\n", name, best, bytes / best / 1e6);
    };
    const int sms = 148;
    run("linear 148x8x256", [&] { k_linear<<<sms * 8, 256>>>(p, n16); });
    for (size_t ch : {512ul, 2048ul, 8192ul, 33792ul, 135168ul}) {
        char nm[64];
        snprintf(nm, 64, "warpchunk %zu B 148x5x256", ch);
        run(nm, [&] { k_warpchunk<<<sms * 5, 256>>>(p, n16, ch / 16); });
    }
    for (size_t ch : {4096ul, 16384ul, 65536ul, 270336ul}) {
        char nm[64];
        snprintf(nm, 64, "blockchunk %zu B 148x5x256", ch);
        run(nm, [&] { k_blockchunk<<<sms * 5, 256>>>(p, n16, ch / 16); });
    }
    {
        const size_t nent = 1030ull << 20;  // ~1.08e9 entries: 4.3 GB + 8.6 GB
        int4 *A, *B;
        cudaFree(p);
        cudaMalloc(&A, nent * 4);
        cudaMalloc(&B, nent * 8);
        for (size_t ch : {2816ul, 11264ul}) {
            char nm[64];
            snprintf(nm, 64, "two arrays 4B+8B, chunk %zu entries", ch);
            cudaEvent_t a2, b2;
            cudaEventCreate(&a2);
            cudaEventCreate(&b2);
            k_two<<<sms * 5, 256>>>(A, B, nent, ch);
            cudaDeviceSynchronize();
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(a2);
                k_two<<<sms * 5, 256>>>(A, B, nent, ch);
                cudaEventRecord(b2);
                cudaEventSynchronize(b2);
                float ms;
                cudaEventElapsedTime(&ms, a2, b2);
                best = ms < best ? ms : best;
            }
            printf("{\"pattern\": \"%s\", \"ms\": %.3f, \"gbs\": %.1f}\n", nm, best, nent * 12.0 / best / 1e6);
        }
    }
    return 0;
}
