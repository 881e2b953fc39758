/*
 * mpxa_device.cuh -- device-side partitioned send (§2.3: "partitioned sends
 * allow so-called early-bird communication ... where partitions are computed in parallel,
 * such as in fork-join parallelism with OpenMP or CUDA kernels").
 *
 * A producer kernel that computes partition i of a partitioned send can publish it the moment
 * it is done, from the device, instead of returning to the host for MPI_Pready:
 *
 *     __global__ void produce(mpxa_psend_dev_t ch, ...) {
 *         int i = blockIdx.x;                       // this CTA computes partition i
 *         ... write partition i of the send buffer ...
 *         __syncthreads();
 *         mpxa_dev_pready(&ch, i);                  // every thread of the CTA calls it
 *     }
 *
 * The handle comes from mpxa_psend_device() (include/mpxa.h) after mpxa_start() of the send
 * request, and stays valid for the request's lifetime.  mpxa_dev_pready copies partition i
 * into the matched receiver's buffer (stores over NVLink when the receiver is on a peer GPU),
 * then release-publishes the partition's arrival flag with the current cycle number.  Each
 * partition must be readied exactly once per cycle, from the device or with the
 * host call mpxa_pready, not both.  The CTA waits (spinning, with the library's watchdog) until
 * the receiver has started the cycle (clear-to-send), so the copy never overwrites data the
 * receiver may still read from the previous cycle.
 *
 * Ownership: the handle's pointers belong to the library; the caller must not free them.
 * Error behaviour: a watchdog expiry sets the comm's error word (mpxa_comm_check() then
 * returns MPXA_ERR_TIMEOUT) and the CTA returns without copying.
 */
#ifndef MPXA_DEVICE_CUH
#define MPXA_DEVICE_CUH

#include <stdint.h>

typedef struct {
    const unsigned char *src;          /* sender buffer (partition i at src + i*part_bytes)   */
    unsigned char *dst;                /* receiver buffer, mapped for this GPU                */
    unsigned long long part_bytes;     /* bytes per sender partition                          */
    int n_parts;                       /* sender partitions                                   */
    int pad;
    unsigned long long *arr;           /* receiver's arrival flags [n_parts] (mapped)         */
    const unsigned long long *cts;     /* cycle the receiver has started (sender memory)      */
    const unsigned long long *scycle;  /* sender's current cycle                              */
    unsigned int *done;                /* per-partition CTA completion counters (sender)      */
    int *err;                          /* comm error word (watchdog)                          */
    long long timeout_ns;
} mpxa_psend_dev_t;

#if defined(__CUDACC__)   /* the struct above is also what host code passes around */
__device__ __forceinline__ unsigned long long mpxa_dev_ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long mpxa_dev_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

/* thread 0 of the calling CTA: spin until *flag >= want; returns 0, or 1 on watchdog expiry */
__device__ __forceinline__ int mpxa_dev_wait_ge(const unsigned long long *flag, unsigned long long want,
                                                int *err, long long timeout_ns) {
    unsigned long long t0 = 0;
    int it = 0;
    while (mpxa_dev_ld_acquire(flag) < want) {
        if (++it > 32) {
            __nanosleep(128);
            if (!t0) t0 = mpxa_dev_now();
            else if ((long long)(mpxa_dev_now() - t0) > timeout_ns) {
                atomicExch(err, 1);
                return 1;
            }
        }
    }
    return 0;
}

/* Copy bytes [lo, hi) of partition i with the threads of this CTA, then, when this CTA is the
 * last of nct CTAs working on partition i, publish its arrival for the current cycle. */
__device__ __forceinline__ void mpxa_dev_pready_part(const mpxa_psend_dev_t *ch, int i, unsigned long long lo,
                                                     unsigned long long hi, unsigned int nct) {
    __shared__ unsigned long long s_cycle;
    __shared__ int s_abort;
    if (threadIdx.x == 0) {
        const unsigned long long cyc = *(volatile const unsigned long long *)ch->scycle;
        s_cycle = cyc;
        s_abort = mpxa_dev_wait_ge(ch->cts, cyc, ch->err, ch->timeout_ns);   /* clear to send */
    }
    __syncthreads();
    if (s_abort) return;
    const unsigned char *s = ch->src + (unsigned long long)i * ch->part_bytes;
    unsigned char *d = ch->dst + (unsigned long long)i * ch->part_bytes;
    const unsigned long long n = hi - lo;
    if ((((uintptr_t)(s + lo) | (uintptr_t)(d + lo) | n) & 15) == 0) {
        const uint4 *s4 = (const uint4 *)(s + lo);
        uint4 *d4 = (uint4 *)(d + lo);
        const unsigned long long nv = n / 16, bd = blockDim.x;
        unsigned long long k = threadIdx.x;
        for (; k + 3 * bd < nv; k += 4 * bd) {      /* four 16-B loads in flight per thread */
            const uint4 a = __ldcg(s4 + k), b = __ldcg(s4 + k + bd), c = __ldcg(s4 + k + 2 * bd),
                        e = __ldcg(s4 + k + 3 * bd);
            d4[k] = a; d4[k + bd] = b; d4[k + 2 * bd] = c; d4[k + 3 * bd] = e;
        }
        for (; k < nv; k += bd) d4[k] = __ldcg(s4 + k);
    } else {
        for (unsigned long long k = lo + threadIdx.x; k < hi; k += blockDim.x) d[k] = (unsigned char)__ldcg(s + k);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        /* Count this CTA's completion with an acq_rel RMW at system scope: the release half
         * publishes the CTA's stores (ordered before it by the barrier), the acquire half lets
         * the last CTA's release below cover every other CTA's stores too (cumulativity) --
         * no separate fence.sc.sys, which costs microseconds. */
        unsigned int prev;
        if (nct == 1u) {
            prev = 0u;
        } else {
            asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&ch->done[i]) : "memory");
        }
        if (prev + 1u == nct) {
            if (nct > 1u) ch->done[i] = 0;   /* every CTA of partition i has counted: reset */
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&ch->arr[i]), "l"(s_cycle) : "memory");
        }
    }
}

/* Early-bird Pready from a producer kernel: the calling CTA copies and publishes partition i. */
__device__ __forceinline__ void mpxa_dev_pready(const mpxa_psend_dev_t *ch, int i) {
    mpxa_dev_pready_part(ch, i, 0, ch->part_bytes, 1u);
}

#endif /* __CUDACC__ */
#endif /* MPXA_DEVICE_CUH */
