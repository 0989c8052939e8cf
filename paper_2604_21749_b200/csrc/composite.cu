// composite.cu — sort-last composite of per-GPU visibility buffers over NCCL
// (NVLink 5 / NVSwitch): unsigned 64-bit min, i.e. ncclMin on ncclUint64.
// The reference composites per-worker buffers with np.minimum
// (pipeline.py:183-204); min is associative and commutative and ties break
// on the global ID, so the composite equals the 1-GPU frame bit for bit.
// Never reduce as int64: CLEAR (all ones) is -1 as a signed value.
//
// Built as a separate library (libcurast_nccl.so) so the rasterizer has no
// NCCL dependency; it binds to whichever libnccl.so.2 the process has loaded
// (torch's), which is API compatible.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static thread_local char g_nerr[256];
static int nfail(ncclResult_t r, const char *where) {
    snprintf(g_nerr, sizeof(g_nerr), "%s: %s", where, ncclGetErrorString(r));
    return -2;
}

extern "C" {

const char *curast_nccl_last_error(void) { return g_nerr; }

int curast_nccl_unique_id(char *out128) {
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return nfail(r, "ncclGetUniqueId");
    memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
    return 0;
}

int curast_nccl_init(void **comm_out, const char *id128, int nranks, int rank) {
    ncclUniqueId id;
    memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm;
    ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) return nfail(r, "ncclCommInitRank");
    *comm_out = (void *)comm;
    return 0;
}

int curast_nccl_destroy(void *comm) {
    ncclResult_t r = ncclCommDestroy((ncclComm_t)comm);
    return r == ncclSuccess ? 0 : nfail(r, "ncclCommDestroy");
}

// every rank ends with the composite frame
int curast_nccl_allreduce_min_u64(void *comm, uint64_t *buf, int64_t n, void *stream) {
    ncclResult_t r = ncclAllReduce(buf, buf, (size_t)n, ncclUint64, ncclMin, (ncclComm_t)comm,
                                   (cudaStream_t)stream);
    return r == ncclSuccess ? 0 : nfail(r, "ncclAllReduce(u64,min)");
}

// root ends with the composite frame
int curast_nccl_reduce_min_u64(void *comm, const uint64_t *send, uint64_t *recv, int64_t n,
                               int root, void *stream) {
    ncclResult_t r = ncclReduce(send, recv, (size_t)n, ncclUint64, ncclMin, root,
                                (ncclComm_t)comm, (cudaStream_t)stream);
    return r == ncclSuccess ? 0 : nfail(r, "ncclReduce(u64,min)");
}

// rank r ends with stripe r (n/nranks words) of the composite frame
int curast_nccl_reduce_scatter_min_u64(void *comm, const uint64_t *send, uint64_t *recv,
                                       int64_t recv_n, void *stream) {
    ncclResult_t r = ncclReduceScatter(send, recv, (size_t)recv_n, ncclUint64, ncclMin,
                                       (ncclComm_t)comm, (cudaStream_t)stream);
    return r == ncclSuccess ? 0 : nfail(r, "ncclReduceScatter(u64,min)");
}

}  // extern "C"
