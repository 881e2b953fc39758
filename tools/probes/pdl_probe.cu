// Probe: the per-launch floor of tiny dependent kernels in a CUDA graph (200 launches back to
// back, one 64-thread CTA moving 16 B): (a) plain launch; (b) programmatic dependent launch
// (PDL) with griddepcontrol.wait at the start and launch_dependents right after; (c) PDL with a
// descriptor load (the kind of table the library reads) before the wait; (d) like (c) with
// 512 threads and 4 KiB of static shared memory.  Prints us per launch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

struct Desc { const uint4 *src; uint4 *dst; };

template <int MODE>
__global__ void k(const Desc *__restrict__ d, const uint4 *src, uint4 *dst) {
    __shared__ uint4 pad[256];
    if (MODE >= 2) {   // descriptor round trip before the dependency wait (overlaps under PDL)
        const Desc dd = d[0];
        src = dd.src;
        dst = dd.dst;
    }
    if (MODE >= 1) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;");
    }
    if (threadIdx.x == 0) {
        uint4 v = __ldcg(src);
        if (MODE == 3) { pad[threadIdx.x] = v; __syncthreads(); v = pad[0]; }
        dst[0] = v;
    } else if (MODE == 3) {
        __syncthreads();
    }
}

template <int MODE>
float run(const Desc *d, const uint4 *s, uint4 *o, cudaStream_t st, int threads) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 200; i++) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(threads);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = MODE >= 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k<MODE>, d, s, o);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best * 1e3f / 200;
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    uint4 *s, *o;
    Desc *d;
    cudaMalloc(&s, 4096);
    cudaMalloc(&o, 4096);
    cudaMalloc(&d, sizeof(Desc));
    Desc h{s, o};
    cudaMemcpy(d, &h, sizeof h, cudaMemcpyHostToDevice);
    printf("(a) plain: %.3f us\n", run<0>(d, s, o, st, 64));
    printf("(b) PDL wait first: %.3f us\n", run<1>(d, s, o, st, 64));
    printf("(c) PDL + descriptor load before the wait: %.3f us\n", run<2>(d, s, o, st, 64));
    printf("(d) as (c), 512 threads + smem + barrier: %.3f us\n", run<3>(d, s, o, st, 512));
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
