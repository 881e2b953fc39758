// Test-only "application" kernel for f3: each CTA computes one partition of a partitioned
// send and publishes it from the device with mpxa_dev_pready (include/mpxa_device.cuh) --
// the early-bird pattern of PAPER.md:160-161.  Built by tests/test_gpu_partitioned.py.
#include <cuda_runtime.h>
#include <string.h>

#include "mpxa_device.cuh"

__global__ void produce_and_pready(mpxa_psend_dev_t ch, unsigned char *buf, int seed) {
    const int i = blockIdx.x;                                  // partition computed by this CTA
    unsigned char *part = buf + (unsigned long long)i * ch.part_bytes;
    for (unsigned long long k = threadIdx.x; k < ch.part_bytes; k += blockDim.x)
        part[k] = (unsigned char)((k * 131u + (unsigned)i * 7u + (unsigned)seed) & 0xff);
    __syncthreads();
    mpxa_dev_pready(&ch, i);
}

extern "C" int launch_produce(const void *handle, int partitions, void *buf, int seed, void *stream) {
    mpxa_psend_dev_t ch;
    memcpy(&ch, handle, sizeof ch);
    produce_and_pready<<<partitions, 256, 0, (cudaStream_t)stream>>>(ch, (unsigned char *)buf, seed);
    return (int)cudaGetLastError();
}
