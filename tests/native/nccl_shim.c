/* nccl_shim.c -- TEST ONLY: a logging stand-in for libnccl.so.2, loaded by
 * libgmg through its GMG_NCCL_LIB dlopen hook (api.cu Nccl::load).  Every
 * communication call is appended to the file named by GMG_SHIM_LOG with
 * "_<rank>" appended; no data moves (sends and receives complete at once,
 * all-reduces leave the buffer as it is), so ranks never wait on one another
 * and several ranks can share one GPU.  tests/test_gpu_nccl_shim.py checks
 * that the recorded sequences of all ranks match pairwise. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef int ncclResult_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef void *ncclComm_t;
typedef int ncclDataType_t;
typedef int ncclRedOp_t;
typedef void *cudaStream_t;

static FILE *logf_ = NULL;
static int rank_ = -1;

static void openlog_(int rank)
{
    if (logf_) return;
    const char *base = getenv("GMG_SHIM_LOG");
    char path[4096];
    snprintf(path, sizeof path, "%s_%d", base ? base : "/tmp/gmg_nccl_shim", rank);
    logf_ = fopen(path, "w");
}

ncclResult_t ncclCommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank)
{
    (void)id;
    rank_ = rank;
    openlog_(rank);
    if (logf_) { fprintf(logf_, "init %d %d\n", nranks, rank); fflush(logf_); }
    *comm = (ncclComm_t)(long)(rank + 1);
    return 0;
}
ncclResult_t ncclCommDestroy(ncclComm_t comm)
{
    (void)comm;
    if (logf_) { fprintf(logf_, "destroy\n"); fclose(logf_); logf_ = NULL; }
    return 0;
}
ncclResult_t ncclGroupStart(void) { if (logf_) fprintf(logf_, "group\n"); return 0; }
ncclResult_t ncclGroupEnd(void) { if (logf_) { fprintf(logf_, "end\n"); fflush(logf_); } return 0; }
ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t s)
{
    (void)buf; (void)c; (void)s;
    if (logf_) fprintf(logf_, "send %d %zu %d\n", peer, count, t);
    return 0;
}
ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t s)
{
    (void)buf; (void)c; (void)s;
    if (logf_) fprintf(logf_, "recv %d %zu %d\n", peer, count, t);
    return 0;
}
ncclResult_t ncclAllReduce(const void *sb, void *rb, size_t count, ncclDataType_t t, ncclRedOp_t op, ncclComm_t c,
                           cudaStream_t s)
{
    (void)sb; (void)rb; (void)c; (void)s;
    if (logf_) { fprintf(logf_, "allreduce %zu %d %d\n", count, t, op); fflush(logf_); }
    return 0;
}
const char *ncclGetErrorString(ncclResult_t r) { (void)r; return "nccl shim"; }
