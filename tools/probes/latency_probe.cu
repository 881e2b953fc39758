// Launch-latency probe (measurement tool): per-launch device time of near-empty kernels in
// a CUDA graph, adding one prologue ingredient of mpxa_exec_kernel at a time.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int V>
__global__ void __launch_bounds__(256, 2) k(int *out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[6];
    if (V >= 1 && threadIdx.x == 0) {
        for (int i = 0; i < 6; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (V >= 2 && threadIdx.x == 0) asm volatile("fence.proxy.async;" ::: "memory");
    if (V >= 3 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (V >= 4) asm volatile("fence.proxy.async;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 999) out[blockIdx.x] = (int)(uintptr_t)sm;
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s failed: %s\n", #x, cudaGetErrorString(e)); fflush(stdout); return -1.f; } } while (0)
static cudaStream_t g_s;
template <typename F>
float graph_time(F launch, int n = 50) {
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(g_s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < n; i++) launch(g_s);
    CK(cudaStreamEndCapture(g_s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0ULL));
    CK(cudaGraphLaunch(ge, g_s)); CK(cudaStreamSynchronize(g_s));
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, g_s)); CK(cudaGraphLaunch(ge, g_s)); CK(cudaEventRecord(b, g_s)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    return ms * 1000 / n;
}
int main() {
    int *out; cudaMalloc(&out, 1 << 20);
    cudaStreamCreate(&g_s);
    printf("start\n"); fflush(stdout);
    const char *names[] = {"empty", "+mbarrier init/fence", "+fence.proxy.async t0", "+bulk wait_group", "+fence.proxy.async all"};
    auto run = [&](void (*kern)(int *), int v) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304);
        for (int smem : {0, 98304}) {
            for (int grid : {1, 8, 148, 296, 1184}) {
                float us = graph_time([&](cudaStream_t s) { kern<<<grid, 256, smem, s>>>(out); });
                printf("%-26s smem %6d grid %5d : %7.2f us/launch\n", names[v], smem, grid, us);
                fflush(stdout);
            }
        }
    };
    run(k<0>, 0); run(k<1>, 1); run(k<2>, 2); run(k<3>, 3); run(k<4>, 4);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
