// Probe: 1-D TMA tensor-map loads from an 8-B-aligned (not 16-B) source offset, with the map
// passed as a __grid_constant__ kernel parameter and used (a) directly, (b) through a pointer
// handed to a __noinline__ function, (c) from a struct member like the executor's TmaMaps.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <vector>

struct Maps { CUtensorMap m[2]; uint64_t base[2]; int elem; int pad[15]; };

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __noinline__ void load(uint32_t dst, const CUtensorMap *map, uint32_t x, uint32_t mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(2048u) : "memory");  // 256 x 8 B
    asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                 ::"r"(dst), "l"((uint64_t)(uintptr_t)map), "r"(x), "r"(mbar) : "memory");
}

template <int MODE>
__global__ void k(const __grid_constant__ Maps M, uint64_t *out, uint32_t x, uint32_t bytes) {
    __shared__ __align__(128) uint64_t buf[256];
    __shared__ __align__(8) uint64_t mbar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&mbar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const CUtensorMap *mp = &M.m[0];
        if (MODE == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&mbar)), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                         ::"r"(su32(buf)), "l"((uint64_t)(uintptr_t)mp), "r"(x), "r"(su32(&mbar)) : "memory");
        } else {
            load(su32(buf), mp, x, su32(&mbar));
        }
        for (long it = 0; it < 100000000; it++) {   // bounded wait (no hang on a wrong tx count)
            uint32_t ok;
            asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n}"
                         : "=r"(ok) : "r"(su32(&mbar)) : "memory");
            if (ok) break;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const size_t n = 1 << 20;
    std::vector<uint64_t> h(n);
    for (size_t i = 0; i < n; i++) h[i] = i * 0x9E3779B97F4A7C15ull;
    uint64_t *d, *out;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&out, 256 * 8);
    cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    Maps M{};
    cuuint64_t gd[1] = {n}, gs[1] = {0};
    cuuint32_t bx[1] = {256}, es[1] = {1};
    CUresult r = enc(&M.m[0], CU_TENSOR_MAP_DATA_TYPE_UINT64, 1, d, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d sizeof(Maps)=%zu\n", (int)r, sizeof(Maps));
    // 4-byte elements: coordinates 2 (8 B), 4 (16 B), 1 (4 B)
    Maps M4{};
    {
        cuuint64_t gd4[1] = {2 * n};
        cuuint32_t bx4[1] = {256};
        CUresult r4 = enc(&M4.m[0], CU_TENSOR_MAP_DATA_TYPE_UINT32, 1, d, gd4, gs, bx4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode4 %d\n", (int)r4);
        for (uint32_t x : {4u, 2u, 1u}) {
            k<0><<<1, 128>>>(M4, out, x, 1024u);
            cudaError_t e = cudaDeviceSynchronize();
            printf("u32 map x %u (byte %u): %s\n", x, 4 * x, cudaGetErrorString(e));
            if (e != cudaSuccess) return 1;
        }
    }
    for (int mode = 0; mode < 2; mode++) {
        for (uint32_t x : {0u, 2u, 12346u, 1u}) {
            cudaMemset(out, 0, 256 * 8);
            if (mode == 0) k<0><<<1, 128>>>(M, out, x, 2048u);
            else k<1><<<1, 128>>>(M, out, x, 2048u);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<uint64_t> o(256);
            cudaMemcpy(o.data(), out, 256 * 8, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int i = 0; i < 256; i++) {
                uint64_t want = x + i < n ? h[x + i] : 0;
                bad += o[i] != want;
            }
            printf("mode %d x %u: %s bad=%d\n", mode, x, cudaGetErrorString(e), bad);
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
