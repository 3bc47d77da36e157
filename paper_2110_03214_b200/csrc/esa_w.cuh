// esa_w.cuh — per-width entry points, included by esa_w{8,16,32}_p{0..4}.cu
// with MAPA_W and MAPA_PART defined: part p < 4 instantiates the single-query
// kernels of base selector p (Greedy / Preserve-insensitive / Preserve-
// sensitive / Baseline), part 4 the batch and trace kernels, so the ~100
// kernel instantiations per width compile as parallel translation units.
#include <atomic>

#include "esa_kernels.cuh"

#define MAPA_CAT2(a, b) a##b
#define MAPA_CAT(a, b) MAPA_CAT2(a, b)

namespace mapa {
namespace {

template <int W, int K, int SEL>
int do_launch_single(const SingleTables &tb, const mapa_query *dq, mapa_record *rec, int D, int rank, int world,
                     int stripe, int grid, cudaStream_t st) {
    const int smem = smem_single(SEL, smem_bytes(tb));
    // the attribute is always set to the fixed upper bound (see kSmemSingleMax),
    // so the occupancy query and every launch agree
    // kernel attributes are per device: one flag bit per device ordinal
    static std::atomic<unsigned long long> configured{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return (int)cudaErrorInvalidDevice;
    if (!((configured.load(std::memory_order_relaxed) >> dev) & 1ull)) {
        cudaError_t e = cudaFuncSetAttribute((const void *)esa_single<W, K, SEL>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemSingleMax);
        if (e != cudaSuccess) return (int)e;
        configured.fetch_or(1ull << dev);
    }
    if (smem > kSmemSingleMax) return (int)cudaErrorInvalidValue;
    esa_single<W, K, SEL><<<grid, kBlock, smem, st>>>(tb, dq, rec, D, rank, world, stripe);
    return (int)cudaGetLastError();
}

using SingleFn = int (*)(const SingleTables &, const mapa_query *, mapa_record *, int, int, int, int, int,
                         cudaStream_t);

// the prune bit (16) applies to k >= 4 only (the host never sets it below)
template <int W, int SEL>
SingleFn pick_k(int K) {
    constexpr int S3 = SEL & ~16, S2 = SEL & ~(16 | 32);  // lin16 from k = 3, prune from k = 4
    switch (K) {
        case 1: return do_launch_single<W, 1, S2>;
        case 2: return do_launch_single<W, 2, S2>;
        case 3: return do_launch_single<W, 3, S3>;
        case 4: return do_launch_single<W, 4, SEL>;
        case 5: return do_launch_single<W, 5, SEL>;
        case 6: return do_launch_single<W, 6, SEL>;
        case 7: return do_launch_single<W, 7, SEL>;
        case 8: return do_launch_single<W, 8, SEL>;
    }
    return nullptr;
}

template <int W, int K, int SEL>
const void *single_ptr() { return (const void *)esa_single<W, K, SEL>; }

template <int W, int SEL>
const void *pick_ptr(int K) {
    constexpr int S3 = SEL & ~16, S2 = SEL & ~(16 | 32);
    switch (K) {
        case 1: return single_ptr<W, 1, S2>();
        case 2: return single_ptr<W, 2, S2>();
        case 3: return single_ptr<W, 3, S3>();
        case 4: return single_ptr<W, 4, SEL>();
        case 5: return single_ptr<W, 5, SEL>();
        case 6: return single_ptr<W, 6, SEL>();
        case 7: return single_ptr<W, 7, SEL>();
        case 8: return single_ptr<W, 8, SEL>();
    }
    return nullptr;
}

// lin16 (bit 5) exists for W = 16 / 32 and the additive selectors only
#define MAPA_SEL_SWITCH(FN, ...)                      \
    if (MAPA_W == 8 || (sc & 3) >= SEL_SENS) sc &= ~32; \
    switch (sc & 55) {                                \
        case 32: return FN<MAPA_W, 32 * (MAPA_W > 8) + 0>(__VA_ARGS__);   \
        case 33: return FN<MAPA_W, 32 * (MAPA_W > 8) + 1>(__VA_ARGS__);   \
        case 36: return FN<MAPA_W, 32 * (MAPA_W > 8) + 4>(__VA_ARGS__);   \
        case 37: return FN<MAPA_W, 32 * (MAPA_W > 8) + 5>(__VA_ARGS__);   \
        case 48: return FN<MAPA_W, 32 * (MAPA_W > 8) + 16>(__VA_ARGS__);  \
        case 49: return FN<MAPA_W, 32 * (MAPA_W > 8) + 17>(__VA_ARGS__);  \
        case 52: return FN<MAPA_W, 32 * (MAPA_W > 8) + 20>(__VA_ARGS__);  \
        case 53: return FN<MAPA_W, 32 * (MAPA_W > 8) + 21>(__VA_ARGS__);  \
        case 0: return FN<MAPA_W, 0>(__VA_ARGS__);    \
        case 1: return FN<MAPA_W, 1>(__VA_ARGS__);    \
        case 2: return FN<MAPA_W, 2>(__VA_ARGS__);    \
        case 3: return FN<MAPA_W, 3>(__VA_ARGS__);    \
        case 4: return FN<MAPA_W, 4>(__VA_ARGS__);    \
        case 5: return FN<MAPA_W, 5>(__VA_ARGS__);    \
        case 6: return FN<MAPA_W, 6>(__VA_ARGS__);    \
        case 7: return FN<MAPA_W, 7>(__VA_ARGS__);    \
        case 16: return FN<MAPA_W, 16>(__VA_ARGS__);  \
        case 17: return FN<MAPA_W, 17>(__VA_ARGS__);  \
        case 18: return FN<MAPA_W, 18>(__VA_ARGS__);  \
        case 19: return FN<MAPA_W, 19>(__VA_ARGS__);  \
        case 20: return FN<MAPA_W, 20>(__VA_ARGS__);  \
        case 21: return FN<MAPA_W, 21>(__VA_ARGS__);  \
        case 22: return FN<MAPA_W, 22>(__VA_ARGS__);  \
        default: return FN<MAPA_W, 23>(__VA_ARGS__);  \
    }

// single-query selector codes compiled into this part (the dispatcher in
// esa.cu routes by sc & 3, so a code outside the part is never asked for)
constexpr bool owns_sel(int sel) { return MAPA_PART < 4 && (sel & 3) == MAPA_PART; }
template <int W, int SEL>
SingleFn pick_k_part(int K) {
    if constexpr (owns_sel(SEL)) return pick_k<W, SEL>(K);
    else return nullptr;
}
template <int W, int SEL>
const void *pick_ptr_part(int K) {
    if constexpr (owns_sel(SEL)) return pick_ptr<W, SEL>(K);
    else return nullptr;
}

SingleFn pick(int K, int sc) { MAPA_SEL_SWITCH(pick_k_part, K) }
const void *pick_fn(int K, int sc) { MAPA_SEL_SWITCH(pick_ptr_part, K) }

}  // namespace

#if MAPA_PART < 4
#define MAPA_PNAME(f) MAPA_CAT(MAPA_CAT(f, MAPA_W), MAPA_CAT(_p, MAPA_PART))
// sc = selector code | 4 * canonical | 16 * prune (SelT)
int MAPA_PNAME(launch_single_w)(const SingleTables &tb, int sc, const mapa_query *dq, mapa_record *rec,
                                      int D, int rank, int world, int stripe, int grid, void *stream) {
    SingleFn fn = pick(tb.pat[0].k, sc);
    if (!fn) return (int)cudaErrorInvalidValue;
    return fn(tb, dq, rec, D, rank, world, stripe, grid, (cudaStream_t)stream);
}

int MAPA_PNAME(occ_single_w)(int K, int sc, int smem) {
    const void *f = pick_fn(K, sc);
    int nb = 0;
    if (!f || set_smem(f, kSmemSingleMax) != 0) return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kBlock, smem_single(sc, smem)) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}
#else

int MAPA_CAT(launch_batch_w, MAPA_W)(const MultiTables &tb, int canon, int64_t nq, const mapa_query *d_queries,
                                     mapa_record *d_results, uint32_t *d_ctr, const uint32_t *d_perm, int grid,
                                     void *stream) {
    const int smem = smem_bytes(tb);
    const void *f = canon ? (const void *)esa_batch<MAPA_W, 1> : (const void *)esa_batch<MAPA_W, 0>;
    int err = set_smem(f, smem);
    if (err) return err;
    if (canon)
        esa_batch<MAPA_W, 1><<<grid, kBlock, smem, (cudaStream_t)stream>>>(tb, (long long)nq, d_queries, d_results,
                                                                         d_ctr, d_perm);
    else
        esa_batch<MAPA_W, 0><<<grid, kBlock, smem, (cudaStream_t)stream>>>(tb, (long long)nq, d_queries, d_results,
                                                                         d_ctr, d_perm);
    return (int)cudaGetLastError();
}

int MAPA_CAT(occ_batch_w, MAPA_W)(int canon, int smem) {
    const void *f = canon ? (const void *)esa_batch<MAPA_W, 1> : (const void *)esa_batch<MAPA_W, 0>;
    int nb = 0;
    if (set_smem(f, smem) != 0) return 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kBlock, smem) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}

int MAPA_CAT(launch_trace_w, MAPA_W)(const MultiTables &tb, int canon, int ntraces, int nops,
                                     const mapa_trace_op *d_ops, int njobs, const mapa_query *d_jobs,
                                     uint64_t *d_keys, void *stream) {
    const int smem = smem_bytes(tb);
    unsigned long long *k = reinterpret_cast<unsigned long long *>(d_keys);
    const void *f = canon ? (const void *)esa_trace<MAPA_W, 1> : (const void *)esa_trace<MAPA_W, 0>;
    int err = set_smem(f, smem);
    if (err) return err;
    if (canon)
        esa_trace<MAPA_W, 1><<<ntraces, kBlock, smem, (cudaStream_t)stream>>>(tb, nops, d_ops, njobs, d_jobs, k);
    else
        esa_trace<MAPA_W, 0><<<ntraces, kBlock, smem, (cudaStream_t)stream>>>(tb, nops, d_ops, njobs, d_jobs, k);
    return (int)cudaGetLastError();
}

int MAPA_CAT(smem_shared_w, MAPA_W)() { return (int)sizeof(Shared); }
#endif

}  // namespace mapa
