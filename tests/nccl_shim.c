/* Test infrastructure: a host-staged stand-in for libnccl.so.2 that lets the
 * library's real multi-rank code (angle sectors, image rows, z-slabs: the
 * ncclAllReduce / ncclSend / ncclRecv / ncclBroadcast call sequences on the
 * session stream)
 * run as several processes on ONE GPU.  Every collective synchronises the
 * caller's stream, copies the device buffer to the host, exchanges it through
 * files in a rendezvous directory (the "unique id" is its path) and copies the
 * result back: ranks wait for each other on the host only, never inside a
 * kernel.  The sum of an allreduce is taken in rank order (((r0 + r1) + r2)
 * ...), which is what the single-device sector emulation computes, so a
 * sharded run can be compared with it bit for bit.  Only the entry points and
 * types the library resolves are provided (float32 / float64 sums).
 *
 *   gcc -O2 -shared -fPIC -I<cuda>/include nccl_shim.c -o libnccl_shim.so -L<cuda>/lib64/stubs -lcuda
 */
#include <cuda.h>
#include <errno.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

typedef struct { char internal[128]; } ncclUniqueId;

typedef struct {
    char dir[112];
    int rank, nranks;
    long ar_seq;
    long *p2p_send, *p2p_recv; /* per peer sequence numbers */
    long* bcast_seq;           /* per root */
} shim_comm;

enum { OP_SEND, OP_RECV, OP_BCAST };
typedef struct {
    int kind;
    void* buf;
    size_t bytes;
    int peer; /* the root of a broadcast */
    shim_comm* comm;
    CUstream stream;
    const void* src; /* broadcast source on the root */
} shim_op;

static shim_op g_ops[4096];
static int g_nops = 0, g_group = 0;

static size_t elem_size(int dtype)
{
    switch (dtype) {
        case 7: return 4; /* float32 */
        case 8: return 8; /* float64 */
        case 0: case 1: return 1;
        case 2: case 3: return 4;
        case 4: case 5: return 8;
        default: return 0;
    }
}

static void wait_file(const char* path)
{
    struct stat st;
    long spins = 0;
    while (stat(path, &st) != 0) {
        usleep(50);
        if (++spins > 300L * 1000 * 1000 / 50) { /* 300 s: a peer is gone */
            fprintf(stderr, "nccl_shim: timeout waiting for %s\n", path);
            abort();
        }
    }
}

static int write_file(const char* path, const void* data, size_t bytes)
{
    char tmp[320];
    snprintf(tmp, sizeof tmp, "%s.part", path);
    FILE* f = fopen(tmp, "wb");
    if (!f) return 1;
    if (bytes && fwrite(data, 1, bytes, f) != bytes) { fclose(f); return 1; }
    fclose(f);
    return rename(tmp, path) != 0; /* readers see whole files only */
}

static int read_file(const char* path, void* data, size_t bytes)
{
    FILE* f = fopen(path, "rb");
    if (!f) return 1;
    size_t got = bytes ? fread(data, 1, bytes, f) : 0;
    fclose(f);
    return got != bytes;
}

int ncclGetUniqueId(ncclUniqueId* id)
{
    memset(id, 0, sizeof *id);
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    const char* base = getenv("PT_NCCL_SHIM_DIR");
    snprintf(id->internal, sizeof id->internal, "%s/shim_%d_%ld_%ld", base ? base : "/tmp",
             (int)getpid(), (long)ts.tv_sec, (long)ts.tv_nsec);
    return mkdir(id->internal, 0700) == 0 ? 0 : 2;
}

int ncclCommInitRank(shim_comm** comm, int nranks, ncclUniqueId id, int rank)
{
    shim_comm* c = (shim_comm*)calloc(1, sizeof *c);
    if (!c) return 1;
    memcpy(c->dir, id.internal, sizeof c->dir - 1);
    c->rank = rank;
    c->nranks = nranks;
    c->p2p_send = (long*)calloc((size_t)nranks, sizeof(long));
    c->p2p_recv = (long*)calloc((size_t)nranks, sizeof(long));
    c->bcast_seq = (long*)calloc((size_t)nranks, sizeof(long));
    *comm = c;
    return 0;
}

int ncclCommDestroy(shim_comm* c)
{
    if (c) {
        free(c->p2p_send);
        free(c->p2p_recv);
        free(c->bcast_seq);
        free(c);
    }
    return 0;
}

const char* ncclGetErrorString(int e)
{
    (void)e;
    return "nccl shim error";
}

int ncclAllReduce(const void* send, void* recv, size_t count, int dtype, int op, shim_comm* c,
                  CUstream stream)
{
    const size_t es = elem_size(dtype);
    if (op != 0 || (dtype != 7 && dtype != 8) || !es) return 5; /* sum of f32 / f64 only */
    const size_t bytes = count * es;
    if (cuStreamSynchronize(stream) != CUDA_SUCCESS) return 1;
    char* mine = (char*)malloc(bytes ? bytes : 1);
    char* acc = (char*)malloc(bytes ? bytes : 1);
    char* other = (char*)malloc(bytes ? bytes : 1);
    if (bytes && cuMemcpyDtoH(mine, (CUdeviceptr)send, bytes) != CUDA_SUCCESS) return 1;
    char path[320];
    snprintf(path, sizeof path, "%s/ar_%ld_%d", c->dir, c->ar_seq, c->rank);
    if (write_file(path, mine, bytes)) return 1;
    for (int r = 0; r < c->nranks; ++r) {
        snprintf(path, sizeof path, "%s/ar_%ld_%d", c->dir, c->ar_seq, r);
        wait_file(path);
        char* dst = r == 0 ? acc : other;
        if (r == c->rank) memcpy(dst, mine, bytes);
        else if (read_file(path, dst, bytes)) return 1;
        if (r == 0) continue;
        if (dtype == 7) {
            float* a = (float*)acc;
            const float* b = (const float*)other;
            for (size_t i = 0; i < count; ++i) a[i] = a[i] + b[i];
        } else {
            double* a = (double*)acc;
            const double* b = (const double*)other;
            for (size_t i = 0; i < count; ++i) a[i] = a[i] + b[i];
        }
    }
    if (bytes && cuMemcpyHtoD((CUdeviceptr)recv, acc, bytes) != CUDA_SUCCESS) return 1;
    /* every rank has read round seq - 1 before anyone writes round seq + 1 */
    if (c->ar_seq >= 1) {
        snprintf(path, sizeof path, "%s/ar_%ld_%d", c->dir, c->ar_seq - 1, c->rank);
        unlink(path);
    }
    ++c->ar_seq;
    free(mine);
    free(acc);
    free(other);
    return 0;
}

static int run_op(const shim_op* o)
{
    char path[320];
    shim_comm* c = o->comm;
    if (o->kind == OP_BCAST) {
        snprintf(path, sizeof path, "%s/bc_%d_%ld", c->dir, o->peer, c->bcast_seq[o->peer]++);
        char* h = (char*)malloc(o->bytes ? o->bytes : 1);
        int rc = 0;
        if (c->rank == o->peer) {
            if (o->bytes && cuMemcpyDtoH(h, (CUdeviceptr)o->src, o->bytes) != CUDA_SUCCESS) rc = 1;
            if (!rc) rc = write_file(path, h, o->bytes);
            if (!rc && o->src != o->buf && o->bytes &&
                cuMemcpyHtoD((CUdeviceptr)o->buf, h, o->bytes) != CUDA_SUCCESS)
                rc = 1;
        } else {
            wait_file(path);
            rc = read_file(path, h, o->bytes);
            if (!rc && o->bytes && cuMemcpyHtoD((CUdeviceptr)o->buf, h, o->bytes) != CUDA_SUCCESS)
                rc = 1;
        }
        free(h);
        return rc;
    }
    if (o->kind == OP_SEND) {
        char* h = (char*)malloc(o->bytes ? o->bytes : 1);
        if (o->bytes && cuMemcpyDtoH(h, (CUdeviceptr)o->buf, o->bytes) != CUDA_SUCCESS) return 1;
        snprintf(path, sizeof path, "%s/p2p_%d_%d_%ld", c->dir, c->rank, o->peer,
                 c->p2p_send[o->peer]++);
        const int rc = write_file(path, h, o->bytes);
        free(h);
        return rc;
    }
    snprintf(path, sizeof path, "%s/p2p_%d_%d_%ld", c->dir, o->peer, c->rank,
             c->p2p_recv[o->peer]++);
    wait_file(path);
    char* h = (char*)malloc(o->bytes ? o->bytes : 1);
    if (read_file(path, h, o->bytes)) return 1;
    unlink(path);
    if (o->bytes && cuMemcpyHtoD((CUdeviceptr)o->buf, h, o->bytes) != CUDA_SUCCESS) return 1;
    free(h);
    return 0;
}

static int flush_ops(void)
{
    /* what this rank publishes first (sends, broadcasts it roots; they never
       block), then what it waits for (receives, the other roots' broadcasts) */
    for (int i = 0; i < g_nops; ++i)
        if (cuStreamSynchronize(g_ops[i].stream) != CUDA_SUCCESS) return 1;
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < g_nops; ++i) {
            const shim_op* o = &g_ops[i];
            const int publishes = o->kind == OP_SEND ||
                                  (o->kind == OP_BCAST && o->comm->rank == o->peer);
            if (publishes == (k == 0) && run_op(o)) return 1;
        }
    g_nops = 0;
    return 0;
}

static int queue_op(int kind, void* buf, size_t count, int dtype, int peer, shim_comm* c,
                    CUstream stream, const void* src)
{
    const size_t es = elem_size(dtype);
    if (!es || g_nops >= (int)(sizeof g_ops / sizeof g_ops[0])) return 5;
    shim_op o = {kind, buf, count * es, peer, c, stream, src};
    g_ops[g_nops++] = o;
    return g_group ? 0 : flush_ops();
}

int ncclSend(const void* buf, size_t count, int dtype, int peer, shim_comm* c, CUstream stream)
{
    return queue_op(OP_SEND, (void*)buf, count, dtype, peer, c, stream, NULL);
}

int ncclRecv(void* buf, size_t count, int dtype, int peer, shim_comm* c, CUstream stream)
{
    return queue_op(OP_RECV, buf, count, dtype, peer, c, stream, NULL);
}

int ncclBroadcast(const void* send, void* recv, size_t count, int dtype, int root, shim_comm* c,
                  CUstream stream)
{
    return queue_op(OP_BCAST, recv, count, dtype, root, c, stream, send);
}

int ncclGroupStart(void)
{
    ++g_group;
    return 0;
}

int ncclGroupEnd(void)
{
    if (g_group > 0 && --g_group == 0) return flush_ops();
    return 0;
}
