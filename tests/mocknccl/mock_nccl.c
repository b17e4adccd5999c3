/*
 * mock_nccl.c -- TEST INFRASTRUCTURE.  A host-mediated stand-in for the
 * handful of NCCL entry points the engine dlopens (ncclGetUniqueId,
 * ncclCommInitRank, ncclCommDestroy, ncclSend, ncclRecv, ncclGroupStart,
 * ncclGroupEnd, ncclAllReduce, ncclGetErrorString), so that the engine's
 * one-shard-per-process code path (halo, window payloads, norm all-reduce,
 * nested chain) runs with several processes on the single GPU a test box has.
 *
 * Transport: every message is copied device->host after synchronising the
 * caller's stream, written to a file under /dev/shm/<id> and renamed into
 * place; receivers poll for the file, read it and copy host->device.  All
 * waiting happens on the host -- no kernel waits on another process -- and a
 * group posts all of its sends before blocking on its receives.  The
 * all-reduce sums (or maxes) the ranks' contributions in rank order.
 * A receive that finds no message within MOCKNCCL_TIMEOUT_MS (default 60 s)
 * fails with ncclSystemError, so a dead peer surfaces as an error the way
 * the engine's timeout does with real NCCL; ncclCommGetAsyncError /
 * ncclCommAbort exist for the engine's fault path.
 *
 * Not used by the product: selected only by tests via ATM_NCCL_LIB.
 */
#include <cuda.h>
#include <dirent.h>
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

typedef enum { ncclSuccess = 0, ncclSystemError = 2, ncclInvalidArgument = 4 } ncclResult_t;
typedef enum { ncclFloat64 = 8 } ncclDataType_t;
typedef enum { ncclSum = 0, ncclMax = 2 } ncclRedOp_t;
typedef struct { char internal[128]; } ncclUniqueId;

typedef struct {
    char dir[128];
    int nranks, rank;
    long* sent;   /* per destination message counters */
    long* recvd;  /* per source message counters */
    long reduce_seq;
} mock_comm;
typedef mock_comm* ncclComm_t;

typedef struct {
    int is_send;
    void* buf;
    size_t bytes;
    int peer;
    mock_comm* comm;
    CUstream stream;
} op_t;

static op_t g_ops[256];
static int g_nops = 0, g_group = 0;

static ncclResult_t fail(const char* what) {
    fprintf(stderr, "mock_nccl: %s (%s)\n", what, strerror(errno));
    return ncclSystemError;
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    memset(id, 0, sizeof(*id));
    struct timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    snprintf(id->internal, sizeof(id->internal), "/dev/shm/mocknccl_%d_%ld_%ld", (int)getpid(),
             (long)ts.tv_sec, (long)ts.tv_nsec);
    if (mkdir(id->internal, 0700) != 0 && errno != EEXIST) return fail("mkdir");
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    mock_comm* c = (mock_comm*)calloc(1, sizeof(mock_comm));
    snprintf(c->dir, sizeof(c->dir), "%s", id.internal);
    mkdir(c->dir, 0700);
    c->nranks = nranks;
    c->rank = rank;
    c->sent = (long*)calloc((size_t)nranks, sizeof(long));
    c->recvd = (long*)calloc((size_t)nranks, sizeof(long));
    *comm = c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
    if (!c) return ncclSuccess;
    free(c->sent);
    free(c->recvd);
    free(c);
    return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
    return r == ncclSuccess ? "success" : "mock transport error (timed out or failed)";
}

ncclResult_t ncclCommGetAsyncError(ncclComm_t c, ncclResult_t* out) {
    (void)c;
    *out = ncclSuccess;  /* every mock operation completes (or fails) synchronously */
    return ncclSuccess;
}

ncclResult_t ncclCommAbort(ncclComm_t c) { return ncclCommDestroy(c); }

static ncclResult_t put_file(const char* path, const void* data, size_t bytes) {
    char tmp[256];
    snprintf(tmp, sizeof(tmp), "%s.tmp", path);
    FILE* f = fopen(tmp, "wb");
    if (!f) return fail("fopen");
    if (bytes && fwrite(data, 1, bytes, f) != bytes) {
        fclose(f);
        return fail("fwrite");
    }
    fclose(f);
    if (rename(tmp, path) != 0) return fail("rename");
    return ncclSuccess;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

static ncclResult_t get_file(const char* path, void* data, size_t bytes) {
    const char* env = getenv("MOCKNCCL_TIMEOUT_MS");
    const double limit = env ? atof(env) : 60000.0, t0 = now_ms();
    for (long spin = 0;; ++spin) {
        FILE* f = fopen(path, "rb");
        if (f) {
            size_t got = bytes ? fread(data, 1, bytes, f) : 0;
            fclose(f);
            if (got != bytes) return fail("short read");
            return ncclSuccess;
        }
        if (now_ms() - t0 > limit) {
            errno = ETIMEDOUT;
            return fail("timed out waiting for a message");
        }
        usleep(50);
    }
}

static ncclResult_t run_send(op_t* o) {
    void* h = malloc(o->bytes ? o->bytes : 1);
    if (cuStreamSynchronize(o->stream) != CUDA_SUCCESS) return fail("stream sync");
    if (o->bytes && cuMemcpyDtoH(h, (CUdeviceptr)o->buf, o->bytes) != CUDA_SUCCESS) return fail("DtoH");
    char path[256];
    snprintf(path, sizeof(path), "%s/p2p_%d_%d_%ld", o->comm->dir, o->comm->rank, o->peer,
             o->comm->sent[o->peer]++);
    ncclResult_t r = put_file(path, h, o->bytes);
    free(h);
    return r;
}

static ncclResult_t run_recv(op_t* o) {
    void* h = malloc(o->bytes ? o->bytes : 1);
    char path[256];
    snprintf(path, sizeof(path), "%s/p2p_%d_%d_%ld", o->comm->dir, o->peer, o->comm->rank,
             o->comm->recvd[o->peer]++);
    ncclResult_t r = get_file(path, h, o->bytes);
    if (r == ncclSuccess) {
        unlink(path);
        /* stream-ordered copy, complete before h is freed: a plain cuMemcpyHtoD
         * from pageable memory may return before its DMA lands, and the
         * engine's non-blocking stream does not order after the null stream */
        if (o->bytes && cuMemcpyHtoDAsync((CUdeviceptr)o->buf, h, o->bytes, o->stream) != CUDA_SUCCESS)
            r = fail("HtoD");
        else if (cuStreamSynchronize(o->stream) != CUDA_SUCCESS) r = fail("stream sync");
    }
    free(h);
    return r;
}

static ncclResult_t flush(void) {
    ncclResult_t r = ncclSuccess;
    for (int i = 0; i < g_nops && r == ncclSuccess; ++i)
        if (g_ops[i].is_send) r = run_send(&g_ops[i]);
    for (int i = 0; i < g_nops && r == ncclSuccess; ++i)
        if (!g_ops[i].is_send) r = run_recv(&g_ops[i]);
    g_nops = 0;
    return r;
}

ncclResult_t ncclGroupStart(void) {
    ++g_group;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd(void) {
    if (--g_group == 0) return flush();
    return ncclSuccess;
}

static ncclResult_t post(int is_send, const void* buf, size_t count, ncclDataType_t t, int peer,
                         ncclComm_t c, CUstream s) {
    if (t != ncclFloat64) return ncclInvalidArgument;
    if (g_nops >= 256) return ncclInvalidArgument;
    op_t o = {is_send, (void*)buf, count * 8, peer, c, s};
    g_ops[g_nops++] = o;
    return g_group ? ncclSuccess : flush();
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c,
                      CUstream s) {
    return post(1, buf, count, t, peer, c, s);
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c,
                      CUstream s) {
    return post(0, buf, count, t, peer, c, s);
}

ncclResult_t ncclAllReduce(const void* sb, void* rb, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t c, CUstream s) {
    if (t != ncclFloat64) return ncclInvalidArgument;
    const size_t bytes = count * 8;
    double* mine = (double*)malloc(bytes ? bytes : 8);
    double* acc = (double*)malloc(bytes ? bytes : 8);
    double* tmp = (double*)malloc(bytes ? bytes : 8);
    if (cuStreamSynchronize(s) != CUDA_SUCCESS) return fail("stream sync");
    if (bytes && cuMemcpyDtoH(mine, (CUdeviceptr)sb, bytes) != CUDA_SUCCESS) return fail("DtoH");
    char path[256];
    const long seq = c->reduce_seq++;
    snprintf(path, sizeof(path), "%s/red_%ld_%d", c->dir, seq, c->rank);
    ncclResult_t r = put_file(path, mine, bytes);
    for (int q = 0; q < c->nranks && r == ncclSuccess; ++q) {
        snprintf(path, sizeof(path), "%s/red_%ld_%d", c->dir, seq, q);
        r = get_file(path, tmp, bytes);
        for (size_t i = 0; i < count && r == ncclSuccess; ++i) {
            if (q == 0) acc[i] = tmp[i];
            else if (op == ncclMax) acc[i] = tmp[i] > acc[i] ? tmp[i] : acc[i];
            else acc[i] += tmp[i];
        }
    }
    if (r == ncclSuccess && bytes &&
        (cuMemcpyHtoDAsync((CUdeviceptr)rb, acc, bytes, s) != CUDA_SUCCESS || cuStreamSynchronize(s) != CUDA_SUCCESS))
        r = fail("HtoD");
    /* files of reduction seq-2 can no longer be read by anyone */
    if (seq >= 2) {
        snprintf(path, sizeof(path), "%s/red_%ld_%d", c->dir, seq - 2, c->rank);
        unlink(path);
    }
    free(mine);
    free(acc);
    free(tmp);
    return r;
}
