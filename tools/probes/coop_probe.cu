// Probe: can a launch carry both the cooperative and the programmatic-stream-serialization
// (PDL) attributes on sm_100a, and what does each cost?  200 dependent launches in a CUDA graph
// of a kernel whose CTAs meet at one grid barrier (a counter, reset by the last CTA) and copy
// 16 B per CTA.  Modes: plain, PDL, cooperative, cooperative + PDL; grids of 1 / 148 / 296 CTAs
// (128 threads).  Prints the launch / capture error codes and us per launch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__global__ void k(unsigned *bar, unsigned *gen, const uint4 *src, uint4 *dst, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        dst[blockIdx.x] = __ldcg(src + blockIdx.x);
        const unsigned g0 = *(volatile unsigned *)gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {   // last arrival releases the others
            *bar = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*(volatile unsigned *)gen == g0) {}
        }
    }
    __syncthreads();
    if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}

static float run(int mode, int nC, unsigned *bar, unsigned *gen, const uint4 *s, uint4 *o, cudaStream_t st,
                 cudaError_t *err) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    *err = cudaSuccess;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 200; i++) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nC);
        cfg.blockDim = dim3(128);
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (mode & 1) {
            at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[na].val.programmaticStreamSerializationAllowed = 1;
            na++;
        }
        if (mode & 2) {
            at[na].id = cudaLaunchAttributeCooperative;
            at[na].val.cooperative = 1;
            na++;
        }
        cfg.attrs = at;
        cfg.numAttrs = na;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k, bar, gen, s, o, (int)(mode & 1));
        if (e != cudaSuccess && *err == cudaSuccess) *err = e;
    }
    cudaError_t ec = cudaStreamEndCapture(st, &g);
    if (*err != cudaSuccess || ec != cudaSuccess) {
        if (*err == cudaSuccess) *err = ec;
        cudaGetLastError();
        return -1.f;
    }
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { *err = cudaGetLastError(); return -1.f; }
    cudaGraphLaunch(ge, st);
    if ((*err = cudaStreamSynchronize(st)) != cudaSuccess) return -1.f;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return best * 1e3f / 200;
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    unsigned *bar, *gen;
    uint4 *s, *o;
    cudaMalloc(&bar, 256);
    cudaMalloc(&gen, 256);
    cudaMemset(bar, 0, 256);
    cudaMemset(gen, 0, 256);
    cudaMalloc(&s, 1 << 16);
    cudaMalloc(&o, 1 << 16);
    const char *names[4] = {"plain", "pdl", "coop", "coop+pdl"};
    for (int nC : {1, 148, 296}) {
        for (int mode = 0; mode < 4; mode++) {
            cudaError_t e;
            const float us = run(mode, nC, bar, gen, s, o, st, &e);
            printf("ctas=%3d %-9s err=%d (%s) us_per_launch=%.3f\n", nC, names[mode], (int)e, cudaGetErrorString(e), us);
        }
    }
    return 0;
}
