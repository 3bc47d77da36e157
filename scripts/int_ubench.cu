// int_ubench.cu -- integer issue / pipe throughput microbenchmark for the
// roofline of the MAPA kernels ("INT32 lanes/SM/clk: measure
// with a microbenchmark").  Every test runs 8 independent dependency chains
// per thread, 64 warps per SM (full occupancy), and reports lane-ops per SM
// per clock: total lane-ops / (SMs x cycles), cycles = the SM clock cycles
// (clock64) elapsed on the slowest CTA.  Each op is pinned with inline PTX /
// intrinsics; `cuobjdump -sass` of this file shows the SASS each test retires
// (IADD3, LOP3, IMAD, VIADDMNMX, VIADDMNMX.S16x2, VIMNMX3, POPC, SHF, PRMT,
// LDS, LDS.128).
//
// Build + run (B200):  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_ubench scripts/int_ubench.cu
//                      ./int_ubench > profiles/r02_int_peaks.json
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

constexpr int kIters = 4096;
constexpr int kChains = 8;
constexpr int kBlock = 256;

enum Op {
    IADD3, LOP3, IMAD, VIADDMNMX, VIADDMNMX16, VIMNMX3, POPC, SHF, PRMT, MIX_ALU_FMA,
    LDS32, LDS128B, LDS16, NOPS
};
static const char *kNames[NOPS] = {"IADD3", "LOP3", "IMAD", "VIADDMNMX", "VIADDMNMX.S16x2", "VIMNMX3", "POPC",
                                   "SHF", "PRMT", "IADD3+IMAD (1:1)", "LDS.32 gather (conflict-free)",
                                   "LDS.128 broadcast", "LDS.U16 gather (conflict-free)"};
// lane-ops (or loads) per chain per iteration
static const int kOpsPerStep[NOPS] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 2, 1, 1, 1};

template <int OP>
__global__ void __launch_bounds__(kBlock) bench(unsigned *out, unsigned long long *cyc, unsigned seed) {
    __shared__ __align__(16) unsigned smem[4096];
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
    const int lane = threadIdx.x & 31;
    unsigned a[kChains];
    if constexpr (OP == LDS32) {  // row r, bank l -> address of row r+1, bank l
        for (int i = threadIdx.x; i < 4096; i += kBlock) smem[i] = sbase + 4u * ((i + 32) & 4095);
        __syncthreads();
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = sbase + 4u * (((c * 13 + (threadIdx.x >> 5) * 7) & 127) * 32 + lane);
    } else if constexpr (OP == LDS128B) {  // 16-B rows; .x = address of the next row
        for (int i = threadIdx.x; i < 1024; i += kBlock) {
            smem[4 * i] = sbase + 16u * ((i + 1) & 1023);
            smem[4 * i + 1] = smem[4 * i + 2] = smem[4 * i + 3] = i;
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = sbase + 16u * ((c * 97 + (threadIdx.x >> 5) * 31) & 1023);
    } else if constexpr (OP == LDS16) {  // u16 entries: row r (64 entries), lane l at entry 2l (bank l)
        unsigned short *h = reinterpret_cast<unsigned short *>(smem);
        for (int i = threadIdx.x; i < 8192; i += kBlock) h[i] = (unsigned short)(sbase + 2u * ((i + 64) & 8191));
        __syncthreads();
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = sbase + 2u * (((c * 13 + (threadIdx.x >> 5) * 7) & 127) * 64 + 2 * lane);
    } else {
        __syncthreads();
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = threadIdx.x * (c + 3) ^ seed;
    }
    const unsigned b = seed * 7u + 1u, d = seed ^ 0x1234u;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if constexpr (OP == IADD3) {  // two PTX adds = one 3-input IADD3
                asm volatile("add.s32 %0, %0, %1;\n\tadd.s32 %0, %0, %2;" : "+r"(a[c]) : "r"(b), "r"(d));
            } else if constexpr (OP == LOP3) {
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b), "r"(d));
            } else if constexpr (OP == IMAD) {
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(b), "r"(d));
            } else if constexpr (OP == VIADDMNMX) {
                a[c] = (unsigned)__viaddmax_s32((int)a[c], (int)b, (int)d);
                asm volatile("" : "+r"(a[c]));
            } else if constexpr (OP == VIADDMNMX16) {
                a[c] = __viaddmax_s16x2(a[c], b, d);
                asm volatile("" : "+r"(a[c]));
            } else if constexpr (OP == VIMNMX3) {
                a[c] = (unsigned)__vimax3_s32((int)a[c], (int)b, (int)d);
                asm volatile("" : "+r"(a[c]));
            } else if constexpr (OP == POPC) {
                asm volatile("popc.b32 %0, %0;" : "+r"(a[c]));
            } else if constexpr (OP == SHF) {
                asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(b), "r"(d));
            } else if constexpr (OP == PRMT) {
                asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(b), "r"(d));
            } else if constexpr (OP == MIX_ALU_FMA) {
                asm volatile("add.s32 %0, %0, %1;\n\tadd.s32 %0, %0, %2;" : "+r"(a[c]) : "r"(b), "r"(d));
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(b), "r"(d));
            } else if constexpr (OP == LDS32) {
                // pointer chase, conflict-free: lane l stays in bank l (no ALU op per load)
                asm volatile("ld.shared.u32 %0, [%0];" : "+r"(a[c]));
            } else if constexpr (OP == LDS128B) {
                // broadcast: every lane reads the same 16 B, the next row's address in .x
                unsigned y, z, w;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%0];" : "+r"(a[c]), "=r"(y), "=r"(z), "=r"(w));
            } else if constexpr (OP == LDS16) {
                asm volatile("ld.shared.u16 %0, [%0];" : "+r"(a[c]));
            }
        }
    }
    const unsigned long long t1 = clock64();
    unsigned r = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) r ^= a[c];
    out[blockIdx.x * kBlock + threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
static void run(int nsm, int dev_clock_khz, bool last) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bench<OP>, kBlock, 0));
    const int grid = nsm * per_sm;
    unsigned *out;
    unsigned long long *cyc;
    CK(cudaMalloc(&out, sizeof(unsigned) * grid * kBlock));
    CK(cudaMalloc(&cyc, sizeof(unsigned long long) * grid));
    bench<OP><<<grid, kBlock>>>(out, cyc, 12345u);  // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    bench<OP><<<grid, kBlock>>>(out, cyc, 777u);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    unsigned long long *h = (unsigned long long *)malloc(sizeof(unsigned long long) * grid);
    CK(cudaMemcpy(h, cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost));
    unsigned long long mx = 0;
    double mean = 0;
    for (int i = 0; i < grid; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        mean += (double)h[i] / grid;
    }
    const double lane_ops = (double)grid * kBlock * kIters * kChains * kOpsPerStep[OP];
    const double per_sm_clk = lane_ops / ((double)nsm * (double)mx);
    const double f_ghz = (double)mx / (ms * 1e6);  // SM clock during the run (cycles of the slowest CTA / event time)
    printf("  {\"op\": \"%s\", \"lane_ops_per_sm_per_clk\": %.2f, \"warp_inst_per_smsp_per_clk\": %.3f, "
           "\"ctas_per_sm\": %d, \"ms\": %.4f, \"clk_ghz_during_run\": %.4f, \"gops_per_s\": %.1f, "
           "\"mean_over_max_cycles\": %.4f}%s\n",
           kNames[OP], per_sm_clk, per_sm_clk / 4.0 / 32.0, per_sm, ms, f_ghz, lane_ops / (ms * 1e-3) / 1e9,
           mean / (double)mx, last ? "" : ",");
    free(h);
    CK(cudaFree(out));
    CK(cudaFree(cyc));
    (void)dev_clock_khz;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    int clk = 0;
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"max_clock_mhz\": %.0f, \"chains_per_thread\": %d, \"iters\": %d,\n"
           " \"block\": %d, \"results\": [\n",
           p.name, p.multiProcessorCount, clk / 1e3, kChains, kIters, kBlock);
    const int n = p.multiProcessorCount;
    run<IADD3>(n, clk, false);
    run<LOP3>(n, clk, false);
    run<IMAD>(n, clk, false);
    run<VIADDMNMX>(n, clk, false);
    run<VIADDMNMX16>(n, clk, false);
    run<VIMNMX3>(n, clk, false);
    run<POPC>(n, clk, false);
    run<SHF>(n, clk, false);
    run<PRMT>(n, clk, false);
    run<MIX_ALU_FMA>(n, clk, false);
    run<LDS32>(n, clk, false);
    run<LDS128B>(n, clk, false);
    run<LDS16>(n, clk, true);
    printf("]}\n");
    return 0;
}
