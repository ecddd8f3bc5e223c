// Read-bandwidth microbenchmark for the depth sweep's streaming structure (scratch tool, not product code).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o stream_read stream_read.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t *b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(b))); }
__device__ __forceinline__ void mexp(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t *b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(sa(b)),
                 "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void *d, const void *s, uint32_t n, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)),
                 "l"(s), "r"(n), "r"(sa(b)) : "memory");
}

// per-warp pipeline: S stages of R rows x 1 KB (rows strided by `rowstride` floats), tiles round-robin
template <int S, int R, int W>
__global__ void __launch_bounds__(W * 32) k_warp(const float *p, long long n, long long rowstride, float *out, int work) {
    extern __shared__ __align__(128) unsigned char sm[];
    float *buf = (float *)sm;                                  // [W][S][R][256]
    uint64_t *bar = (uint64_t *)(sm + W * S * R * 1024);       // [W][S]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long ntiles = n / 256, stride = (long long)gridDim.x * W;
    long long t = blockIdx.x * W + w;
    if (lane == 0) for (int s = 0; s < S; ++s) minit(&bar[w * S + s]);
    __syncwarp();
    auto issue = [&](int s, long long tt) {
        if (lane == 0 && tt < ntiles) {
            mexp(&bar[w * S + s], R * 1024);
            for (int r = 0; r < R; ++r) bulk(buf + ((w * S + s) * R + r) * 256, p + r * rowstride + tt * 256, 1024, &bar[w * S + s]);
        }
    };
    for (int s = 0; s < S; ++s) issue(s, t + s * stride);
    float acc = 0.f;
    uint32_t ph = 0;
    for (int k = 0;; ++k) {
        const int s = k % S;
        const long long tt = t + (long long)k * stride;
        if (tt >= ntiles) break;
        mwait(&bar[w * S + s], (ph >> s) & 1); ph ^= 1u << s;
        for (int r = 0; r < R; ++r) {
            const float4 v = *(const float4 *)(buf + ((w * S + s) * R + r) * 256 + 4 * lane);
            acc += v.x + v.y + v.z + v.w;
        }
        for (int i = 0; i < work; ++i) acc = fmaf(acc, 1.0000001f, 0.5f);  // emulated per-tile compute
        __syncwarp();
        issue(s, tt + (long long)S * stride);
    }
    if (acc == 123.f) out[0] = acc;
}

// plain vectorised loads, U float4 per thread in flight
template <int U>
__global__ void __launch_bounds__(256) k_ldg(const float4 *p, long long n4, float *out) {
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n4; i += stride * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = i + u * stride < n4 ? __ldcs(p + i + u * stride) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 123.f) out[0] = acc;
}

int main() {
    const long long n = 100000000LL;  // points; 4 rows (x, y, z, r) -> 1.6 GB
    float *p, *out;
    cudaMalloc(&p, 4 * n * sizeof(float));
    cudaMalloc(&out, 64);
    cudaMemset(p, 0, 4 * n * sizeof(float));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](const char *name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(a);
        const int it = 20;
        for (int i = 0; i < it; ++i) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= it;
        printf("%-44s %8.1f us  %6.0f GB/s  %s\n", name, ms * 1e3, 16.0 * n / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    auto warp_cfg = [&](auto kern, int S, int R, int W, int per_sm, int work, const char *name) {
        size_t smem = (size_t)W * S * R * 1024 + W * S * 8;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W * 32, smem);
        int g = sms * (per_sm < occ ? per_sm : occ);
        char nm[128];
        snprintf(nm, sizeof nm, "%s occ=%d work=%d", name, per_sm < occ ? per_sm : occ, work);
        timeit(nm, [&] { kern<<<g, W * 32, smem>>>(p, n, n, out, work); });
    };
    for (int work : {0, 40, 80}) {
        warp_cfg(k_warp<2, 4, 8>, 2, 4, 8, 3, work, "warp S2 R4 W8 x3");
        warp_cfg(k_warp<3, 4, 8>, 3, 4, 8, 2, work, "warp S3 R4 W8 x2");
        warp_cfg(k_warp<4, 4, 4>, 4, 4, 4, 3, work, "warp S4 R4 W4 x3");
        warp_cfg(k_warp<2, 4, 16>, 2, 4, 16, 1, work, "warp S2 R4 W16 x1");
        warp_cfg(k_warp<2, 4, 4>, 2, 4, 4, 6, work, "warp S2 R4 W4 x6");
    }
    timeit("ldg U1 grid sms*8", [&] { k_ldg<1><<<sms * 8, 256>>>((const float4 *)p, n, out); });
    timeit("ldg U4 grid sms*8", [&] { k_ldg<4><<<sms * 8, 256>>>((const float4 *)p, n, out); });
    timeit("ldg U8 grid sms*4", [&] { k_ldg<8><<<sms * 4, 256>>>((const float4 *)p, n, out); });
    return 0;
}
