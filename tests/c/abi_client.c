/* A plain C client of the mpxa C ABI (include/mpxa.h): no Python, no torch.  One process
 * hosting p ranks on one GPU runs the BASELINE cfg1-shaped alltoall (pairwise and Bruck), an
 * allgather and a persistent alltoallv (init once, 5 start/wait cycles) on buffers it
 * allocates with the CUDA runtime, and writes every received buffer to a file for the test
 * to compare with the oracle.  Usage: abi_client <input file> <output file>; the input holds
 * p, b and the send buffers (see tests/test_gpu_c_client.py). */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mpxa.h"

#define CHK(x)                                                                 \
    do {                                                                       \
        int rc_ = (int)(x);                                                    \
        if (rc_) {                                                             \
            fprintf(stderr, "%s failed: %d (%s)\n", #x, rc_, mpxa_error_string(rc_)); \
            return 1;                                                          \
        }                                                                      \
    } while (0)
#define CUCHK(x)                                                               \
    do {                                                                       \
        cudaError_t e_ = (x);                                                  \
        if (e_ != cudaSuccess) {                                               \
            fprintf(stderr, "%s failed: %s\n", #x, cudaGetErrorString(e_));   \
            return 1;                                                          \
        }                                                                      \
    } while (0)

int main(int argc, char **argv) {
    if (argc != 3) return 2;
    FILE *in = fopen(argv[1], "rb");
    if (!in) return 2;
    int64_t hdr[2];
    if (fread(hdr, 8, 2, in) != 2) return 2;
    const int p = (int)hdr[0];
    const size_t b = (size_t)hdr[1];
    const size_t a2a_bytes = (size_t)p * p * b, ag_bytes = (size_t)p * b;
    unsigned char *h_a2a = malloc(a2a_bytes), *h_ag = malloc(ag_bytes), *h_out = malloc(a2a_bytes);
    int64_t *sc = malloc(8 * p * p), *sd = malloc(8 * p * p), *rc = malloc(8 * p * p), *rd = malloc(8 * p * p);
    if (fread(h_a2a, 1, a2a_bytes, in) != a2a_bytes || fread(h_ag, 1, ag_bytes, in) != ag_bytes) return 2;
    if (fread(sc, 8, (size_t)p * p, in) != (size_t)p * p) return 2;
    fclose(in);
    /* alltoallv: packed displacements, recvcounts = transpose (elements of 8 bytes) */
    int64_t smax = 0, rmax = 0;
    for (int r = 0; r < p; r++) {
        int64_t so = 0, ro = 0;
        for (int j = 0; j < p; j++) {
            sd[r * p + j] = so;
            so += sc[r * p + j];
            rc[r * p + j] = sc[j * p + r];
            rd[r * p + j] = ro;
            ro += rc[r * p + j];
        }
        if (so > smax) smax = so;
        if (ro > rmax) rmax = ro;
    }
    const size_t vsb = (size_t)(smax ? smax : 1) * 8, vrb = (size_t)(rmax ? rmax : 1) * 8;

    mpxa_init_args a;
    memset(&a, 0, sizeof a);
    a.nprocs = 1;
    a.proc = 0;
    a.ranks_per_proc = p;
    a.device = 0;
    mpxa_comm_t comm;
    CHK(mpxa_init(&comm, &a));
    int np = 0;
    CHK(mpxa_comm_size(comm, &np));
    if (np != p) return 3;
    cudaStream_t st;
    CUCHK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    void *d_s, *d_r, *d_vs, *d_vr;
    CUCHK(cudaMalloc(&d_s, a2a_bytes));
    CUCHK(cudaMalloc(&d_r, a2a_bytes));
    CUCHK(cudaMalloc(&d_vs, (size_t)p * vsb));
    CUCHK(cudaMalloc(&d_vr, (size_t)p * vrb));
    FILE *out = fopen(argv[2], "wb");
    /* alltoall, pairwise then Bruck (BASELINE cfg1 variants) */
    const mpxa_algo_t algos[2] = {MPXA_ALGO_PAIRWISE, MPXA_ALGO_BRUCK};
    for (int k = 0; k < 2; k++) {
        CUCHK(cudaMemcpy(d_s, h_a2a, a2a_bytes, cudaMemcpyHostToDevice));
        CUCHK(cudaMemset(d_r, 0, a2a_bytes));
        CHK(mpxa_alltoall_algo(d_s, b, 1, d_r, algos[k], comm, (mpxa_stream_t)st));
        CUCHK(cudaStreamSynchronize(st));
        CUCHK(cudaMemcpy(h_out, d_r, a2a_bytes, cudaMemcpyDeviceToHost));
        fwrite(h_out, 1, a2a_bytes, out);
    }
    /* allgather, default variant */
    CUCHK(cudaMemcpy(d_s, h_ag, ag_bytes, cudaMemcpyHostToDevice));
    CUCHK(cudaMemset(d_r, 0, a2a_bytes));
    CHK(mpxa_allgather(d_s, b, 1, d_r, comm, (mpxa_stream_t)st));
    CUCHK(cudaStreamSynchronize(st));
    CUCHK(cudaMemcpy(h_out, d_r, a2a_bytes, cudaMemcpyDeviceToHost));
    fwrite(h_out, 1, a2a_bytes, out);
    /* persistent alltoallv: init once, 5 start / wait cycles; send rows from the a2a input */
    unsigned char *h_vs = calloc((size_t)p, vsb);
    for (int r = 0; r < p; r++)
        for (size_t x = 0; x < vsb; x++) h_vs[(size_t)r * vsb + x] = h_a2a[((size_t)r * vsb + x) % a2a_bytes];
    CUCHK(cudaMemcpy(d_vs, h_vs, (size_t)p * vsb, cudaMemcpyHostToDevice));
    CUCHK(cudaMemset(d_vr, 0xA5, (size_t)p * vrb));
    mpxa_request_t req;
    CHK(mpxa_alltoallv_init(d_vs, sc, sd, vsb, d_vr, rc, rd, vrb, 8, MPXA_ALGO_DEFAULT, comm, NULL, &req));
    for (int cyc = 0; cyc < 5; cyc++) {
        CHK(mpxa_start(req, (mpxa_stream_t)st));
        CHK(mpxa_wait(req, (mpxa_stream_t)st));
    }
    CUCHK(cudaStreamSynchronize(st));
    unsigned char *h_vr = malloc((size_t)p * vrb);
    CUCHK(cudaMemcpy(h_vr, d_vr, (size_t)p * vrb, cudaMemcpyDeviceToHost));
    const int64_t dims[2] = {(int64_t)vsb, (int64_t)vrb};
    fwrite(dims, 8, 2, out);
    fwrite(h_vs, 1, (size_t)p * vsb, out);
    fwrite(h_vr, 1, (size_t)p * vrb, out);
    fclose(out);
    CHK(mpxa_request_free(&req));
    CHK(mpxa_comm_check(comm));
    uint64_t launches = 0;
    CHK(mpxa_launch_count(comm, &launches));
    printf("launches %llu\n", (unsigned long long)launches);
    CHK(mpxa_finalize(comm));
    return 0;
}
