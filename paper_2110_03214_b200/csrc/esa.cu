// esa.cu — host dispatch of the Enumerate-Score-Argmax kernels by topology
// width W (8 / 16 / 32); the kernels themselves are in esa_kernels.cuh and are
// instantiated per W and part by esa_w{8,16,32}_p{0..4}.cu (see esa_w.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace mapa {

#define MAPA_DECL_P(W, P)                                                                                       \
    int launch_single_w##W##_p##P(const SingleTables &, int, const mapa_query *, mapa_record *, int, int, int, int, \
                                  int, void *);                                                                     \
    int occ_single_w##W##_p##P(int, int, int);
#define MAPA_DECL_W(W)                                                                                       \
    MAPA_DECL_P(W, 0) MAPA_DECL_P(W, 1) MAPA_DECL_P(W, 2) MAPA_DECL_P(W, 3)                                   \
    int launch_batch_w##W(const MultiTables &, int, int64_t, const mapa_query *, mapa_record *, uint32_t *,  \
                          const uint32_t *, int, void *);                                                    \
    int occ_batch_w##W(int, int);                                                                            \
    int launch_trace_w##W(const MultiTables &, int, int, int, const mapa_trace_op *, int, const mapa_query *, \
                          uint64_t *, void *);                                                               \
    int smem_shared_w##W();
MAPA_DECL_W(8)
MAPA_DECL_W(16)
MAPA_DECL_W(32)

// single-query kernels live in per-selector parts (esa_w*_p<sc & 3>.cu)
#define MAPA_SINGLE_PARTS(W, FN, ...)                      \
    switch (sc & 3) {                                      \
        case 0: return FN##_w##W##_p0(__VA_ARGS__);        \
        case 1: return FN##_w##W##_p1(__VA_ARGS__);        \
        case 2: return FN##_w##W##_p2(__VA_ARGS__);        \
        default: return FN##_w##W##_p3(__VA_ARGS__);       \
    }

int launch_single(const SingleTables &tb, int sc, const mapa_query *d_query, mapa_record *d_record, int depth,
                  int rank, int world, int stripe, int grid, void *stream) {
    switch (tb.topo.width) {
        case 8: MAPA_SINGLE_PARTS(8, launch_single, tb, sc, d_query, d_record, depth, rank, world, stripe, grid, stream)
        case 16: MAPA_SINGLE_PARTS(16, launch_single, tb, sc, d_query, d_record, depth, rank, world, stripe, grid, stream)
        case 32: MAPA_SINGLE_PARTS(32, launch_single, tb, sc, d_query, d_record, depth, rank, world, stripe, grid, stream)
    }
    return (int)cudaErrorInvalidValue;
}

int launch_batch(const MultiTables &tb, int canon, int64_t nq, const mapa_query *d_queries, mapa_record *d_results,
                 uint32_t *d_ctr, const uint32_t *d_perm, int grid, void *stream) {
    switch (tb.topo.width) {
        case 8: return launch_batch_w8(tb, canon, nq, d_queries, d_results, d_ctr, d_perm, grid, stream);
        case 16: return launch_batch_w16(tb, canon, nq, d_queries, d_results, d_ctr, d_perm, grid, stream);
        case 32: return launch_batch_w32(tb, canon, nq, d_queries, d_results, d_ctr, d_perm, grid, stream);
    }
    return (int)cudaErrorInvalidValue;
}

namespace {

// Code path of a batch query: (k - 1) * 4 + selector code (32 buckets; a bad
// pattern index goes to bucket 0 and is flagged by the batch kernel).
__device__ __forceinline__ int bucket_of(const mapa_query &q, const BucketKeys &bk) {
    if (q.pattern >= (uint32_t)bk.npats) return 0;
    return ((int)bk.k[q.pattern] - 1) * 4 + sel_code(q.selector, q.sensitive);
}

// Pass 1: per-bucket counts (warp-aggregated atomics).
__global__ void bucket_count(BucketKeys bk, long long nq, const mapa_query *__restrict__ qs,
                             unsigned int *__restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nq; base += stride) {
        const long long q = base + lane;
        const int key = q < nq ? bucket_of(qs[q], bk) : 32;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
        if (key < 32 && lane == __ffs(peers) - 1) atomicAdd(&cnt[key], (unsigned)__popc(peers));
    }
}

// Pass 2: scatter query indices to their bucket's slice of perm (order inside
// a bucket is arbitrary; results do not depend on it).
__global__ void bucket_scatter(BucketKeys bk, long long nq, const mapa_query *__restrict__ qs,
                               const unsigned int *__restrict__ cnt, unsigned int *__restrict__ cursor,
                               uint32_t *__restrict__ perm) {
    __shared__ unsigned int start[33];
    if (threadIdx.x < 32) {
        const unsigned c = cnt[threadIdx.x];
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if ((int)threadIdx.x >= o) incl += v;
        }
        start[threadIdx.x] = incl - c;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < nq; base += stride) {
        const long long q = base + lane;
        const int key = q < nq ? bucket_of(qs[q], bk) : 32;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
        const int leader = __ffs(peers) - 1;
        unsigned off = 0;
        if (key < 32 && lane == leader) off = atomicAdd(&cursor[key], (unsigned)__popc(peers));
        off = __shfl_sync(0xFFFFFFFFu, off, leader);
        if (key < 32) perm[start[key] + off + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)q;
    }
}

}  // namespace

int launch_bucket(const BucketKeys &bk, int64_t nq, const mapa_query *d_queries, unsigned int *d_cnt,
                  unsigned int *d_cursor, uint32_t *d_perm, void *stream) {
    const int grid = (int)std::min<int64_t>(1184, (nq + 255) / 256);
    if (grid <= 0) return 0;
    bucket_count<<<grid, 256, 0, (cudaStream_t)stream>>>(bk, (long long)nq, d_queries, d_cnt);
    bucket_scatter<<<grid, 256, 0, (cudaStream_t)stream>>>(bk, (long long)nq, d_queries, d_cnt, d_cursor, d_perm);
    return (int)cudaGetLastError();
}

int launch_trace(const MultiTables &tb, int canon, int ntraces, int nops, const mapa_trace_op *d_ops, int njobs,
                 const mapa_query *d_jobs, uint64_t *d_keys, void *stream) {
    switch (tb.topo.width) {
        case 8: return launch_trace_w8(tb, canon, ntraces, nops, d_ops, njobs, d_jobs, d_keys, stream);
        case 16: return launch_trace_w16(tb, canon, ntraces, nops, d_ops, njobs, d_jobs, d_keys, stream);
        case 32: return launch_trace_w32(tb, canon, ntraces, nops, d_ops, njobs, d_jobs, d_keys, stream);
    }
    return (int)cudaErrorInvalidValue;
}

int device_sm_count() {
    // cached per device (host launch path latency: no attribute query per call)
    static int cached[64] = {0};
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    if (dev >= 0 && dev < 64) cached[dev] = n;
    return n;
}

static int occ_single_parts(int width, int k, int sc, int smem) {
    if (width == 8) { MAPA_SINGLE_PARTS(8, occ_single, k, sc, smem) }
    if (width == 16) { MAPA_SINGLE_PARTS(16, occ_single, k, sc, smem) }
    MAPA_SINGLE_PARTS(32, occ_single, k, sc, smem)
}

int max_blocks_per_sm_single(int width, int k, int sc, int xs) {
    // cached: (width, k, selector code with canon bit, xs) -> blocks per SM
    static int cache[3][9][56][48] = {};
    const int wi = width == 8 ? 0 : (width == 16 ? 1 : 2), xi = xs < 48 ? xs : 0;
    int &slot = cache[wi][k >= 1 && k <= 8 ? k : 0][sc & 55][xi];
    if (slot) return slot;
    const int smem = smem_shared_w32() + 4 * xs * xs * (int)sizeof(int);
    int r;
    r = occ_single_parts(width, k, sc, smem);
    slot = r;
    return r;
}

int max_blocks_per_sm_batch(int width, int canon, int npats, int xs) {
    const int smem = smem_shared_w32() + (npats * 3 + 1) * xs * xs * (int)sizeof(int);
    if (width == 8) return occ_batch_w8(canon, smem);
    if (width == 16) return occ_batch_w16(canon, smem);
    return occ_batch_w32(canon, smem);
}

const char *cuda_error_string(int err) { return cudaGetErrorString((cudaError_t)err); }

}  // namespace mapa
