// K4 — composition of affine slice maps y -> G y + c.
//
//  * CHAIN (bit-exact): compose_sweep (nievergelt.cpp:90-110) walking the slices in order; the
//    owner of row i accumulates sum_k G(i,k) y_k sequentially in k exactly like matvec
//    (linalg.cpp:17-26), then adds c_i. For n <= 512: a cluster of ceil(n/32) single-warp CTAs,
//    CTA r owning rows 32r..32r+31 (lane = row); each CTA's 32-row block of the next two maps is
//    bulk-copied into shared memory ahead of use (the block is contiguous in the row-major map),
//    and the new y is exchanged through distributed shared memory with one cluster barrier per
//    map; up to n = 512 with the non-portable cluster sizes (16 CTAs, one 32-row block each).
//    Larger n: one CTA, rows read from global.
//  * TREE (EXTENSION, north_star subsystem 3): log-depth pairwise products
//        (G2, c2) o (G1, c1) = (G2 G1, G2 c1 + c2)
//    on FP64 tensor cores: mma.sync m8n8k4 f64 (SASS DMMA) with 64x64 CTA tiles staged through
//    bank-conflict-free padded shared memory. Tolerance vs the chain: <= 1e-12 relative.
//
// Maps are the row-major augmented blocks [G | c] with leading dimension ldm (pint_cuda.h).
// Roofline: TREE is FP64 tensor (2 n^3 flops per pair); CHAIN is latency/L2 bound.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "pint_internal.cuh"

namespace cg = cooperative_groups;

namespace {

using namespace pint_async;

constexpr int kChainThreads = 256;
// a concurrent chain that gave up waiting (PINT_E_SERIALIZED): above every task and range-retry
// index, so a real failure of the same run is the one reported first
constexpr long long kSerializedIndex = 0x7FFFFFFFFFFFFFFEll;

// One CTA; thread t owns rows t, t+256, ... Dynamic smem: y[n].
__global__ void __launch_bounds__(kChainThreads)
affine_chain_kernel(long long n, long long N, long long ldm, const double* __restrict__ maps,
                    const double* __restrict__ y0, double* __restrict__ y) {
    extern __shared__ double y_s[];
    for (long long i = threadIdx.x; i < n; i += kChainThreads) y_s[i] = y0[i];
    __syncthreads();
    const long long n4 = n / 4;
    for (long long j = 0; j < N; ++j) {
        const double* M = maps + j * n * ldm;
        if (j + 1 < N)  // pull this thread's rows of the next map into L1 while this one is applied
            for (long long i = threadIdx.x; i < n; i += kChainThreads) {
                const char* nxt = reinterpret_cast<const char*>(M + n * ldm + i * ldm);
                for (long long b = 0; b < 8 * (n + 1); b += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(nxt + b));
            }
        double out[4];
        int cnt = 0;
        for (long long i = threadIdx.x; i < n; i += kChainThreads, ++cnt) {
            const double* row = M + i * ldm;
            const double4* row4 = reinterpret_cast<const double4*>(row);
            double s = 0.0;
#pragma unroll 4
            for (long long q = 0; q < n4; ++q) {
                const double4 g = row4[q];
                s = __dadd_rn(s, __dmul_rn(g.x, y_s[4 * q + 0]));
                s = __dadd_rn(s, __dmul_rn(g.y, y_s[4 * q + 1]));
                s = __dadd_rn(s, __dmul_rn(g.z, y_s[4 * q + 2]));
                s = __dadd_rn(s, __dmul_rn(g.w, y_s[4 * q + 3]));
            }
            for (long long k = 4 * n4; k < n; ++k) s = __dadd_rn(s, __dmul_rn(row[k], y_s[k]));
            if (cnt < 4) out[cnt] = __dadd_rn(s, row[n]);
        }
        __syncthreads();
        cnt = 0;
        for (long long i = threadIdx.x; i < n && cnt < 4; i += kChainThreads, ++cnt) y_s[i] = out[cnt];
        __syncthreads();
    }
    for (long long i = threadIdx.x; i < n; i += kChainThreads) y[i] = y_s[i];
}

// Cluster chain (n <= 512). Dynamic smem: rows[ring][32][ldm] | y[2][ny] | pad | ring map barriers
// | 2 y barriers,
// ny = n rounded up to 16 (16-byte aligned y pairs; the pipeline may read 16 doubles past n). A
// CTA's 32 rows of a map are one contiguous block: one bulk copy per map.
constexpr int kClusterMax = 16;  // (> 8: the non-portable cluster sizes, one 32-row block per SM up to n = 512)
constexpr int kChainAhead = 8;  // pairs of terms in flight per lane
constexpr int kRing = 4;        // maps in flight (bulk-copy latency ~ 2 map applications); fewer
                                // when 4 blocks of 32 rows do not fit (n > ~220)

__global__ void __launch_bounds__(32) affine_chain_cluster_kernel(int n, long long N, int ldm, int ring,
                                                                  const double* __restrict__ maps,
                                                                  const double* __restrict__ y0,
                                                                  double* __restrict__ y, const int* ready,
                                                                  int target, FailRec* fail) {
    extern __shared__ __align__(16) double sm[];
    // waiting on builders launched behind this grid on the same stream (programmatic dependent
    // launch): let them start now that this CTA is resident
    if (ready) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    const unsigned csize = cluster.num_blocks();
    const int lane = threadIdx.x;
    const int r0 = 32 * static_cast<int>(rank), rows = min(32, n - r0);
    const int ny = (n + 15) & ~15;
    double* blk = sm;                       // [ring][32][ldm]
    double* ys = sm + ring * 32 * ldm;        // [2][ny] + look-ahead pad
    const unsigned bar0 = smem_u32(ys + 2 * ny + 4 * kChainAhead);  // ring map barriers
    const unsigned ybar0 = bar0 + 8u * ring;                           // 2 y barriers
    const long long mstride = static_cast<long long>(n) * ldm;
    const unsigned blk_bytes = 8u * static_cast<unsigned>(ldm) * static_cast<unsigned>(rows);
    if (lane == 0) {
        for (int b = 0; b < ring + 2; ++b) mbar_init(bar0 + 8u * b);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    const bool mine = lane < rows;
    bool gave_up = false;
    // (ready: maps arrive while this kernel runs — wait until map j's builders have all stored it,
    // then order that acquire before the bulk copy's async-proxy read)
    auto fetch = [&](long long j, int b) {  // this CTA's rows of map j (contiguous) into block b
        if (lane == 0 && ready && !gave_up) {
            int v;
            const unsigned long long t0 = pint_dev::globaltimer();
            do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(ready + j) : "memory");
                // never hang: a map not ready 1 s after the wait began means its builder is not
                // running; fail loudly (the result is not used) and stop waiting for the rest
                if (v < target && pint_dev::globaltimer() - t0 > 1000000000ull) {
                    pint_dev::record_failure(fail, kSerializedIndex, PINT_E_SERIALIZED, static_cast<double>(j));
                    gave_up = true;
                    break;
                }
            } while (v < target);
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
        }
        if (lane == 0)
            bulk_load(smem_u32(blk + b * 32 * ldm), maps + j * mstride + static_cast<long long>(r0) * ldm, blk_bytes,
                      bar0 + 8u * b);
    };
    for (long long j = 0; j < ring && j < N; ++j) fetch(j, static_cast<int>(j));
    for (int i = lane; i < 2 * ny + 4 * kChainAhead; i += 32) ys[i] = (i < n) ? y0[i] : 0.0;
    cluster.sync();  // every CTA's barriers and y buffers are initialised before any remote write
    const int pairs = n / 2;
#ifdef PINT_CHAIN_PROF
    long long tw = 0, tc = 0, tf = 0, ts = 0, t0 = clock64();
#define CHAIN_MARK(v)                   \
    do {                                \
        const long long t1 = clock64(); \
        v += t1 - t0;                   \
        t0 = t1;                        \
    } while (0)
#else
#define CHAIN_MARK(v) \
    do {              \
    } while (0)
#endif
    for (long long j = 0; j < N; ++j) {
        const int b = static_cast<int>(j % ring), yb = static_cast<int>(j & 1);
        mbar_wait(bar0 + 8u * b, static_cast<unsigned>((j / ring) & 1));
        // the block after the ring's next into L2 now, so its bulk copy (issued once this block is
        // consumed) reads L2 rather than HBM — with a 1-deep ring (n > ~220) that copy is exposed
        if (lane == 0 && j + ring < N && (!ready || *reinterpret_cast<const volatile int*>(ready + j + ring) >= target))
            prefetch_l2(maps + (j + ring) * mstride + static_cast<long long>(r0) * ldm, blk_bytes);
        CHAIN_MARK(tw);
        const double2* g2 = reinterpret_cast<const double2*>(blk + (b * 32 + lane) * ldm);
        const double2* y2 = reinterpret_cast<const double2*>(ys + yb * ny);
        double s = 0.0;
        // sum_k G(i,k) y_k in k order (matvec), loads kChainAhead pairs ahead of the DADD chain
        double2 gv[kChainAhead], yv[kChainAhead];
#pragma unroll
        for (int u = 0; u < kChainAhead; ++u) gv[u] = g2[u], yv[u] = y2[u];
        int q = 0;
#pragma unroll 1
        for (; q + kChainAhead <= pairs; q += kChainAhead) {
#pragma unroll
            for (int u = 0; u < kChainAhead; ++u) {
                s = __dadd_rn(s, __dmul_rn(gv[u].x, yv[u].x));
                s = __dadd_rn(s, __dmul_rn(gv[u].y, yv[u].y));
                gv[u] = g2[q + u + kChainAhead];
                yv[u] = y2[q + u + kChainAhead];
            }
        }
#pragma unroll
        for (int u = 0; u < kChainAhead - 1; ++u)
            if (q + u < pairs) {
                s = __dadd_rn(s, __dmul_rn(gv[u].x, yv[u].x));
                s = __dadd_rn(s, __dmul_rn(gv[u].y, yv[u].y));
            }
        const double* g = blk + (b * 32 + lane) * ldm;
        if (n & 1) s = __dadd_rn(s, __dmul_rn(g[n - 1], ys[yb * ny + n - 1]));
        s = __dadd_rn(s, g[n]);  // + c_i
        CHAIN_MARK(tc);
        __syncwarp();  // block b fully read: refill it with map j + ring
        if (j + ring < N) fetch(j + ring, b);
        // y_{j+1}: every CTA's rows land in every CTA's buffer yb^1 via st.async, each completing
        // its bytes on that CTA's y barrier (n * 8 bytes expected per map)
        const unsigned ybar = ybar0 + 8u * (yb ^ 1);
        if (lane == 0)
            asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(ybar),
                         "r"(8u * static_cast<unsigned>(n))
                         : "memory");
        if (mine) {
            const unsigned la = smem_u32(ys + (yb ^ 1) * ny + r0 + lane);
            for (unsigned c = 0; c < csize; ++c) {
                unsigned ra, rb;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(c));
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(ybar), "r"(c));
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(ra),
                             "d"(s), "r"(rb)
                             : "memory");
            }
        }
        CHAIN_MARK(tf);
        mbar_wait(ybar, static_cast<unsigned>((j >> 1) & 1));  // y_{j+1} complete here
        CHAIN_MARK(ts);
    }
#ifdef PINT_CHAIN_PROF
    if (lane == 0)
        printf("rank %u: per map wait %lld compute %lld fetch+store %lld sync %lld cycles\n", rank, tw / N, tc / N,
               tf / N, ts / N);
#endif
    if (mine) y[r0 + lane] = ys[(N & 1) * ny + r0 + lane];
    if (ready && rank == 0 && lane == 0)  // (the span words behind the counters: chain end)
        reinterpret_cast<unsigned long long*>(const_cast<int*>(ready) + ((N + 1) & ~1ll))[2] = pint_dev::globaltimer();
    cluster.sync();  // no CTA leaves while a peer may still write into its shared memory
}

// ---- the WIDE chain: 32 W rows per CTA, maps streamed by TMA (n in (256, 512], n % 16 == 0) -----
// Bit-exact like the cluster chain above (lane = row, sum_k G(i,k) y_k sequential in k, then + c_i).
// A CTA's 32W x (n+1) block does not sit in shared memory, so each consumer warp streams its 32 rows
// through a ring of 16 KB boxes: the maps seen as a 4-D tensor {16 columns, n rows, n/16 column
// blocks, N maps} (strides 8 B, 8 ldm B, 128 B, 8 n ldm B), box {16, 32, 4, 1} = 64 columns x 32
// rows with the 128-byte swizzle, so lane = row reads its 16-byte pairs conflict-free. One producer
// warp issues every box (full/empty mbarrier pairs per slot); the consumers only wait, sum and
// release, loading one 8-pair group ahead of the DADD chain. Beside the exact build W = 4 (4 SMs at
// n = 512 instead of 16: the build gets 144), see launch_affine_chain_on.
constexpr int kWideBlk = 4, kWideCols = 16 * kWideBlk, kWideRingTotal = 12;
constexpr int kWideSlot = 32 * kWideCols;  // doubles

template <int kWideWarps>
__global__ void __launch_bounds__(32 * (kWideWarps + 1)) affine_chain_wide_kernel(
    const __grid_constant__ CUtensorMap tm, int n, long long N, int ldm, const double* __restrict__ maps,
    const double* __restrict__ y0, double* __restrict__ y, const int* ready, int target, FailRec* fail) {
    constexpr int kRows = 32 * kWideWarps, kRing = kWideRingTotal / kWideWarps;
    extern __shared__ __align__(1024) double sm_raw[];
    if (ready) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    // (1024-byte alignment for the swizzled boxes, by offsetting sm_raw itself: the pointer stays a
    // shared-window pointer, so the row reads compile to LDS, not generic loads)
    double* sm = sm_raw + ((((smem_u32(sm_raw) + 1023u) & ~1023u) - smem_u32(sm_raw)) >> 3);
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ny = (n + kWideCols - 1) / kWideCols * kWideCols;
    const int nch = (n + kWideCols - 1) / kWideCols;
    // [warps][kRing][kWideBlk][32 rows][16] | y [2][ny] | full [warps][kRing] | empty [..] | 2 y barriers
    double* ys = sm + kWideWarps * kRing * kWideSlot;
    const unsigned full0 = smem_u32(ys + 2 * ny), empty0 = full0 + 8u * kWideWarps * kRing;
    const unsigned ybar0 = empty0 + 8u * kWideWarps * kRing;
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2 * kWideWarps * kRing + 2; ++b) mbar_init(full0 + 8u * b);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    for (int i = threadIdx.x; i < 2 * ny; i += blockDim.x) ys[i] = (i < n) ? y0[i] : 0.0;
    cluster.sync();  // barriers and y initialised everywhere before any copy lands or remote write
    const long long total = N * nch;
    if (warp == kWideWarps) {  // ---- the producer: lane 0 issues every box of every consumer warp
        if (lane == 0) {
            bool gave_up = false;
            long long j = 0;
            int c = 0, slot = 0;
            unsigned use = 0;  // uses of `slot` so far
            for (long long q = 0; q < total; ++q) {
                if (c == 0 && ready && !gave_up) {  // map j must be complete (its builders counted)
                    int v;
                    const unsigned long long t0 = pint_dev::globaltimer();
                    do {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(ready + j) : "memory");
                        if (v < target && pint_dev::globaltimer() - t0 > 1000000000ull) {
                            pint_dev::record_failure(fail, kSerializedIndex, PINT_E_SERIALIZED, static_cast<double>(j));
                            gave_up = true;
                            break;
                        }
                    } while (v < target);
                    asm volatile("fence.proxy.async.global;\n" ::: "memory");
                }
                for (int w = 0; w < kWideWarps; ++w) {
                    const int row0 = static_cast<int>(rank) * kRows + 32 * w;
                    if (row0 >= n) break;
                    const unsigned fb = full0 + 8u * (w * kRing + slot), eb = empty0 + 8u * (w * kRing + slot);
                    if (use > 0) mbar_wait(eb, (use - 1) & 1);  // the consumer released the slot
                    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(fb),
                                 "r"(8u * kWideSlot)
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
                        "{%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(sm + (w * kRing + slot) * kWideSlot)),
                        "l"(reinterpret_cast<unsigned long long>(&tm)), "r"(0), "r"(row0), "r"(c * kWideBlk),
                        "r"(static_cast<int>(j)), "r"(fb)
                        : "memory");
                }
                if (++slot == kRing) slot = 0, ++use;
                if (++c == nch) c = 0, ++j;
            }
        }
    } else {  // ---- consumers: lane = row
        const int row0 = static_cast<int>(rank) * kRows + warp * 32, row = row0 + lane;
        const bool mine = row < n;
        const double* ring = sm + warp * kRing * kWideSlot + lane * 16;
        const unsigned wfull = full0 + 8u * warp * kRing, wempty = empty0 + 8u * warp * kRing;
// the 128-byte swizzle: 16-byte chunk i of row r sits at chunk i ^ (r & 7) of its 128-byte line
        int off[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) off[u] = 2 * (u ^ (lane & 7));
        int slot = 0;
        unsigned use = 0;
#ifdef PINT_CHAIN_PROF
        long long tb = 0, tyw = 0, tcp = 0, tst = 0, tp = clock64();
#define WMARK(v) do { const long long t1 = clock64(); v += t1 - tp; tp = t1; } while (0)
#else
#define WMARK(v) do { } while (0)
#endif
        for (long long j = 0; j < N; ++j) {
            const int yb = static_cast<int>(j & 1);
            const double2* y2 = reinterpret_cast<const double2*>(ys + yb * ny);
            double s = 0.0;
            if (row0 < n) {
                // the map's n/2 column pairs in order, in 8-pair groups (a 16-column block of a box),
                // each group's operands loaded during the previous group's DADDs. The box loop is
                // straight-line (a warp issues in order: branches between groups would serialise the
                // integer work with the DADD chain); a box's slot is released once it is summed.
                const double* cur = ring + slot * kWideSlot;
                WMARK(tcp);
                mbar_wait(wfull + 8u * slot, use & 1);
                WMARK(tb);
                // c_i once map j's first box has landed: the producer acquired map j before issuing
                // it, and the barrier's phase carries that here (the build writes c: an L2 load)
                const double cc =
                    mine ? __ldcg(maps + j * static_cast<long long>(n) * ldm + static_cast<long long>(row) * ldm + n) : 0.0;
                double2 gv[8], yq[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) gv[u] = *reinterpret_cast<const double2*>(cur + off[u]), yq[u] = y2[u];
                for (int c = 0; c < nch; ++c) {
                    const int nb = min(kWideBlk, (n - c * kWideCols) / 16);  // 16-column blocks in box c
                    int nslot = slot + 1;
                    unsigned nuse = use;
                    if (nslot == kRing) nslot = 0, ++nuse;
                    const double* nxt = ring + nslot * kWideSlot;
                    const bool more = c + 1 < nch;
                    const double2* yc = y2 + c * (kWideCols / 2);
                    if (nb == kWideBlk) {  // a full box: 4 groups, straight-line
#pragma unroll
                        for (int b = 0; b < kWideBlk; ++b) {
                            if (b == kWideBlk - 1 && more) {
                                WMARK(tcp);
                                mbar_wait(wfull + 8u * nslot, nuse & 1);
                                WMARK(tb);
                            }
                            const double* gn = b + 1 < kWideBlk ? cur + (b + 1) * 32 * 16 : nxt;
                            const double2* yn = yc + (b + 1) * 8;
                            const bool ld = b + 1 < kWideBlk || more;
#pragma unroll
                            for (int u = 0; u < 8; ++u) {  // matvec order: k sequential
                                s = __dadd_rn(s, __dmul_rn(gv[u].x, yq[u].x));
                                s = __dadd_rn(s, __dmul_rn(gv[u].y, yq[u].y));
                                if (ld) gv[u] = *reinterpret_cast<const double2*>(gn + off[u]), yq[u] = yn[u];
                            }
                        }
                    } else {  // the last, partial box (n % 64 != 0)
                        for (int b = 0; b < nb; ++b) {
                            const bool ld = b + 1 < nb;
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                s = __dadd_rn(s, __dmul_rn(gv[u].x, yq[u].x));
                                s = __dadd_rn(s, __dmul_rn(gv[u].y, yq[u].y));
                                if (ld)
                                    gv[u] = *reinterpret_cast<const double2*>(cur + (b + 1) * 32 * 16 + off[u]),
                                    yq[u] = yc[(b + 1) * 8 + u];
                            }
                        }
                    }
                    __syncwarp();  // box c is summed: hand its slot back to the producer
                    if (lane == 0)
                        asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(wempty + 8u * slot)
                                     : "memory");
                    slot = nslot, use = nuse, cur = nxt;
                }
                s = __dadd_rn(s, cc);  // + c_i
            }
            WMARK(tcp);
            // y_{j+1}: every CTA's rows land in every CTA's buffer yb ^ 1 (8n bytes expected per map)
            const unsigned ybar = ybar0 + 8u * (yb ^ 1);
            if (threadIdx.x == 0)
                asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(ybar),
                             "r"(8u * static_cast<unsigned>(n))
                             : "memory");
            if (mine) {
                const unsigned la = smem_u32(ys + (yb ^ 1) * ny + row);
                for (unsigned cc2 = 0; cc2 < csize; ++cc2) {
                    unsigned ra, rb;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(cc2));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(ybar), "r"(cc2));
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(ra),
                                 "d"(s), "r"(rb)
                                 : "memory");
                }
            }
            WMARK(tst);
            mbar_wait(ybar, static_cast<unsigned>((j >> 1) & 1));  // y_{j+1} complete here
            WMARK(tyw);
        }
#ifdef PINT_CHAIN_PROF
        if (lane == 0 && (rank == 0 || rank == csize - 1))
            printf("wide rank %u warp %d: per map box-wait %lld compute %lld send %lld y-wait %lld cycles\n", rank, warp,
                   tb / N, tcp / N, tst / N, tyw / N);
#endif
#undef WMARK
        if (mine) y[row] = ys[(N & 1) * ny + row];
        if (ready && rank == 0 && threadIdx.x == 0)  // (the span words behind the counters: chain end)
            reinterpret_cast<unsigned long long*>(const_cast<int*>(ready) + ((N + 1) & ~1ll))[2] = pint_dev::globaltimer();
    }
    cluster.sync();  // no CTA leaves while a peer may still write into its shared memory
}

// ---- DMMA pair kernel ------------------------------------------------------------------------
// CTA = 2 x 2 warps, warp tile (8 MI) x 32: BM = 16 MI rows, BN = 64 columns (+ the extra fragment).
constexpr int BN = 64, BK = 16, kStages = 3;
constexpr int AS = BK + 4;       // padded strides: conflict-free fragment loads
constexpr int BW = BN + 8;       // B tile width: 64 columns + one 8-column fragment for column n
constexpr int BS = BW + 4;
template <int MI>
constexpr size_t pair_smem_bytes() { return sizeof(double) * kStages * (16 * MI * AS + BK * BS); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// out_p = later_p o earlier_p for pair p = blockIdx.z, as ONE product of augmented matrices:
// [G2 | c2] [[G1, c1], [0, 1]] = [G2 G1 | G2 c1 + c2] — the B tiles span E's n+1 columns (c1 is
// column n) and the epilogue adds c2 to column n. Column tiles cover n columns; when n is a
// multiple of 64 the column n would open a 64-wide tile of its own, so the last tile's right-hand
// warps carry one extra 8-column fragment instead.
template <int MI>
__global__ void __launch_bounds__(128)
affine_pair_kernel(long long n, long long ldm, const double* __restrict__ earlier,
                   long long e_stride, const double* __restrict__ later, long long l_stride,
                   double* __restrict__ out, long long o_stride) {
    constexpr int BM = 16 * MI;
    const long long p = blockIdx.z;
    const double* E = earlier + p * e_stride;
    const double* L = later + p * l_stride;
    double* O = out + p * o_stride;
    const long long row0 = static_cast<long long>(blockIdx.y) * BM;
    const int tid = threadIdx.x;
    const long long nc = n + 1;  // output / B columns

    // kStages-deep cp.async pipeline of BMx16 (A) and 16x72 (B) tiles; out-of-range elements are
    // zero-filled by the copy itself (src-size 0 or 8 of 16)
    extern __shared__ __align__(16) double pair_smem[];
    double* As = pair_smem;                        // [kStages][BM * AS]
    double* Bs = pair_smem + kStages * BM * AS;    // [kStages][BK * BS]
    const long long col0 = static_cast<long long>(blockIdx.x) * BN;
    const int lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const int g = lane >> 2, t4 = lane & 3;

    double acc[MI][5][2];
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
        for (int b = 0; b < 5; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    const bool extra = wn == 1 && col0 + BN == n;  // this warp also owns columns n .. n+7

    auto cp16 = [](double* dst, const double* src, long long bytes) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                     "r"(static_cast<unsigned>(bytes))
                     : "memory");
    };
    auto issue = [&](int stage, long long k0) {
#pragma unroll
        for (int u = 0; u < MI; ++u) {  // A: BM x 16 = 8 MI x 128 16-byte chunks
            const int idx = tid + u * 128;
            const int ar = idx >> 3, ac = (idx & 7) * 2;
            const long long gr = row0 + ar, gc = k0 + ac;
            const long long abytes = gr < n ? 8 * max(0ll, min(2ll, n - gc)) : 0;
            cp16(As + stage * BM * AS + ar * AS + ac, abytes ? L + gr * ldm + gc : L, abytes);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // B: 16 x 64
            const int idx = tid + u * 128;
            const int br = idx >> 5, bc = (idx & 31) * 2;
            const long long gk = k0 + br, gn = col0 + bc;
            const long long bbytes = gk < n ? 8 * max(0ll, min(2ll, nc - gn)) : 0;
            cp16(Bs + stage * BK * BS + br * BS + bc, bbytes ? E + gk * ldm + gn : E, bbytes);
        }
        if (tid < 64) {  // B columns 64..71 of the tile (16 rows x 4 chunks)
            const int br = tid >> 2, bc = BN + (tid & 3) * 2;
            const long long gk = k0 + br, gn = col0 + bc;
            const long long bbytes = gk < n ? 8 * max(0ll, min(2ll, nc - gn)) : 0;
            cp16(Bs + stage * BK * BS + br * BS + bc, bbytes ? E + gk * ldm + gn : E, bbytes);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    const long long kTiles = (n + BK - 1) / BK;
#pragma unroll
    for (int st = 0; st < kStages - 1; ++st) {
        if (st < kTiles) issue(st, st * BK);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    for (long long kt = 0; kt < kTiles; ++kt) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(kStages - 2) : "memory");  // tile kt has landed
        __syncthreads();  // ... for every thread; and stage (kt-1) % kStages is free again
        if (kt + kStages - 1 < kTiles) issue(static_cast<int>((kt + kStages - 1) % kStages), (kt + kStages - 1) * BK);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        const double* A = As + (kt % kStages) * BM * AS;
        const double* B = Bs + (kt % kStages) * BK * BS;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[MI], bf[4];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) af[mi] = A[(wm * 8 * MI + mi * 8 + g) * AS + kk + t4];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) bf[ni] = B[(kk + t4) * BS + wn * 32 + ni * 8 + g];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
            if (extra) {
                const double bx = B[(kk + t4) * BS + BN + g];
#pragma unroll
                for (int mi = 0; mi < MI; ++mi) dmma(acc[mi][4][0], acc[mi][4][1], af[mi], bx);
            }
        }
    }
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
        const long long r = row0 + wm * 8 * MI + mi * 8 + g;
        if (r >= n) continue;
#pragma unroll
        for (int ni = 0; ni < 5; ++ni) {
            if (ni == 4 && !extra) continue;
            const long long c = ni == 4 ? col0 + BN + t4 * 2 : col0 + wn * 32 + ni * 8 + t4 * 2;
            double v0 = acc[mi][ni][0], v1 = acc[mi][ni][1];
            if (c == n) v0 += L[r * ldm + n];          // + c2
            else if (c + 1 == n) v1 += L[r * ldm + n];
            if (c + 1 < nc) {
                *reinterpret_cast<double2*>(O + r * ldm + c) = make_double2(v0, v1);
            } else if (c < nc) {
                O[r * ldm + c] = v0;
            }
        }
    }
}

// ---- DMMA pair kernel, TMA-fed (16 | n) ---------------------------------------------------------
// The same augmented product out_p = later_p o earlier_p, CTA tile 128 x 128 (8 warps of 64 x 32;
// thread 0 also issues the copies), k tiles of 16 in a kPairStages-deep ring filled by TMA with full /
// empty mbarriers — no per-thread address arithmetic and no __syncthreads in the k loop (the
// cp.async kernel above spends as many integer instructions on its copies as it issues DMMAs).
//  * A (later, rows x k): 3-D tensor {n, n, pairs}, box {16 k, 128 rows} with the 128-byte swizzle:
//    row r's 16-byte chunk i at i ^ (r & 7).
//  * B (earlier, k x columns): 4-D tensor {16 columns, n rows, n/16 column blocks, pairs}, box
//    {16, 16, 8, 1} = [8 column blocks][16 k][16 columns], swizzled per 128-byte k line.
//  * the translation column (c1 = earlier's column n) for the last column tile: a {8, 16} box of
//    the {n+1, n, pairs} tensor (columns past n zero-filled), unswizzled.
//  A k step uses k offsets {0, 1, 4, 5} (+ 0, 2, 8, 10) for the four k lanes instead of 0..3: the
//  fragment reads then touch each bank twice (2 wavefronts, the minimum) for A and for B — with
//  consecutive k, B's four rows XOR into the same half of the 128-byte line (4 wavefronts).
constexpr int kPairStages = 4;  // (a power of 2)
constexpr unsigned kPairA = 128 * 16 * 8, kPairB = 8 * 16 * 16 * 8, kPairX = 16 * 8 * 8;  // bytes per stage
constexpr unsigned kPairStage = kPairA + kPairB + kPairX;
struct PairMaps {
    CUtensorMap a, b, x;
};
constexpr size_t pair_tma_smem() { return 1024 + kPairStages * kPairStage + 16 * kPairStages; }

__global__ void __launch_bounds__(256, 1)
affine_pair_tma_kernel(const __grid_constant__ PairMaps tm, int n, long long ldm, int pairs,
                       const double* __restrict__ later, long long l_stride, double* __restrict__ out,
                       long long o_stride, int chunked) {
    extern __shared__ __align__(1024) unsigned char pt_raw[];
    unsigned char* sm = pt_raw + ((((smem_u32(pt_raw) + 1023u) & ~1023u) - smem_u32(pt_raw)));
    const unsigned base = smem_u32(sm);
    const unsigned full0 = base + kPairStages * kPairStage, empty0 = full0 + 8 * kPairStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kTiles = (n + 15) / 16, tiles1 = (n + 127) / 128;
    const int tiles = pairs * tiles1 * tiles1;
    // this CTA's tiles (a contiguous run, see launch_pairs_tma): their k tiles form one sequence
    // q = (local tile) * kTiles + kt through the ring, so the next tile's first stages load while
    // this one's epilogue stores
    // chunked (the default): CTA b takes tiles [b*tiles/grid, (b+1)*tiles/grid); else round-robin
    const int c_lo = static_cast<int>(static_cast<long long>(blockIdx.x) * tiles / gridDim.x);
    const int c_hi = static_cast<int>(static_cast<long long>(blockIdx.x + 1) * tiles / gridDim.x);
    const int my_tiles = chunked ? c_hi - c_lo : blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long total_q = static_cast<long long>(my_tiles) * kTiles;
    struct Tile {
        int p, row0, col0;
        bool xtile;
    };
    auto tile_of = [&](int lt) {
        const int t = chunked ? c_lo + lt : blockIdx.x + lt * gridDim.x;
        Tile T;
        T.p = t / (tiles1 * tiles1);
        const int r = t - T.p * tiles1 * tiles1;
        T.row0 = (r / tiles1) * 128;
        T.col0 = (r % tiles1) * 128;
        T.xtile = T.col0 + 128 >= n;  // the tile holding the last columns also computes column n
        return T;
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPairStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(full0 + 8 * s) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;\n" ::"r"(empty0 + 8 * s) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // thread 0 also feeds the ring: step q into stage q % kPairStages once every warp has released
    // the stage's previous step (a 9th, producer warp would cap the registers at 168: 3 warps on
    // one SM sub-partition)
    // (the producer walks its own (tile, k tile) cursor: no 64-bit divisions on thread 0, whose warp
    // every other warp waits for through the ring)
    long long pq = 0;
    int pkt = 0, plt = 0;
    Tile PT = tile_of(0);
    auto produce_next = [&]() {
        const int s = static_cast<int>(pq & (kPairStages - 1));
        if (pq >= kPairStages) mbar_wait(empty0 + 8 * s, static_cast<unsigned>((pq / kPairStages) - 1) & 1);
        const unsigned fb = full0 + 8 * s, dst = base + s * kPairStage;
        asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(fb),
                     "r"(kPairA + kPairB + (PT.xtile ? kPairX : 0u))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
            "%3, %4}], [%5];\n" ::"r"(dst),
            "l"(reinterpret_cast<unsigned long long>(&tm.a)), "r"(16 * pkt), "r"(PT.row0), "r"(PT.p), "r"(fb)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
            "%3, %4, %5}], [%6];\n" ::"r"(dst + kPairA),
            "l"(reinterpret_cast<unsigned long long>(&tm.b)), "r"(0), "r"(16 * pkt), "r"(PT.col0 / 16), "r"(PT.p),
            "r"(fb)
            : "memory");
        if (PT.xtile)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
                "{%2, %3, %4}], [%5];\n" ::"r"(dst + kPairA + kPairB),
                "l"(reinterpret_cast<unsigned long long>(&tm.x)), "r"(n), "r"(16 * pkt), "r"(PT.p), "r"(fb)
                : "memory");
        ++pq;
        if (++pkt == kTiles) {
            pkt = 0;
            if (++plt < my_tiles) PT = tile_of(plt);
        }
    };
    if (threadIdx.x == 0)
        while (pq < kPairStages && pq < total_q) produce_next();
    // warp (wm, wn) owns rows wm*64 .. +63, columns wn*32 .. +31 of a tile
    const int wm = warp >> 2, wn = warp & 3;
    const int g = lane >> 2, t4 = lane & 3;
    const int kofs = (t4 & 1) + 4 * (t4 >> 1);  // k lane -> k offset {0, 1, 4, 5}
    long long q = 0;
    for (int lt = 0; lt < my_tiles; ++lt) {
        const Tile T = tile_of(lt);
        const bool extra = T.xtile && wn == 3;  // + the 8-column fragment holding column n
        double acc[8][5][2];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 5; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        for (int kt = 0; kt < kTiles; ++kt, ++q) {
            const int s = static_cast<int>(q & (kPairStages - 1));
            mbar_wait(full0 + 8 * s, static_cast<unsigned>(q / kPairStages) & 1);
            const unsigned char* As = sm + s * kPairStage;
            const unsigned char* Bs = As + kPairA;
            const double* Xs = reinterpret_cast<const double*>(Bs + kPairB);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {  // k = kb + kofs, kb in {0, 2, 8, 10}
                const int k = 2 * (ks & 1) + 8 * (ks >> 1) + kofs;
                double af[8], bf[4];
#pragma unroll
                for (int mi = 0; mi < 8; ++mi) {  // A[row][k]: row & 7 == g
                    const int r = wm * 64 + mi * 8 + g;
                    af[mi] = *reinterpret_cast<const double*>(As + r * 128 + (((k >> 1) ^ g) << 4) + ((k & 1) << 3));
                }
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) {  // B[k][c]: block c / 16, k line, chunk (c & 15) / 2 ^ (k & 7)
                    const int c = wn * 32 + ni * 8 + g;
                    bf[ni] = *reinterpret_cast<const double*>(Bs + (c >> 4) * 2048 + k * 128 +
                                                              ((((c & 15) >> 1) ^ (k & 7)) << 4) + ((c & 1) << 3));
                }
#pragma unroll
                for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
                if (extra) {
                    const double bx = Xs[k * 8 + g];
#pragma unroll
                    for (int mi = 0; mi < 8; ++mi) dmma(acc[mi][4][0], acc[mi][4][1], af[mi], bx);
                }
            }
            __syncwarp();
            if (lane == 0)
                asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(empty0 + 8 * s)
                             : "memory");
            if (threadIdx.x == 0 && pq < total_q) produce_next();
        }
        const double* L = later + T.p * l_stride;
        double* O = out + T.p * o_stride;
        const long long nc = n + 1;
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) {
            const long long r = T.row0 + wm * 64 + mi * 8 + g;
            if (r >= n) continue;
#pragma unroll
            for (int ni = 0; ni < 5; ++ni) {
                if (ni == 4 && !extra) continue;
                const long long c = ni == 4 ? n + t4 * 2 : T.col0 + wn * 32 + ni * 8 + t4 * 2;
                if (ni < 4 && c >= n) continue;
                double v0 = acc[mi][ni][0], v1 = acc[mi][ni][1];
                if (c == n) v0 += L[r * ldm + n];  // + c2
                if (c + 1 < n) {
                    *reinterpret_cast<double2*>(O + r * ldm + c) = make_double2(v0, v1);
                } else if (c < nc) {
                    O[r * ldm + c] = v0;
                }
            }
        }
    }
}

int launch_pairs_tma(pint_ctx* ctx, long long n, long long P, const double* earlier, long long e_stride,
                     const double* later, long long l_stride, double* out, long long o_stride) {
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(pint_tensor_map_encoder());
    if (!enc) return pint_set_error(ctx, PINT_E_CUDA, "affine_pair: cuTensorMapEncodeTiled unavailable");
    const long long ldm = pint_affine_ldm(n);
    PairMaps M;
    const cuuint32_t e1[4] = {1, 1, 1, 1};
    {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(P)};
        const cuuint64_t str[2] = {static_cast<cuuint64_t>(8 * ldm), static_cast<cuuint64_t>(8 * l_stride)};
        const cuuint32_t box[3] = {16, 128, 1};
        if (enc(&M.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(later), dims, str, box, e1,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return pint_set_error(ctx, PINT_E_CUDA, "affine_pair: tensor map A failed");
    }
    {
        const cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(n / 16),
                                    static_cast<cuuint64_t>(P)};
        const cuuint64_t str[3] = {static_cast<cuuint64_t>(8 * ldm), 128, static_cast<cuuint64_t>(8 * e_stride)};
        const cuuint32_t box[4] = {16, 16, 8, 1};
        if (enc(&M.b, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(earlier), dims, str, box, e1,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return pint_set_error(ctx, PINT_E_CUDA, "affine_pair: tensor map B failed");
    }
    {
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(n + 1), static_cast<cuuint64_t>(n),
                                    static_cast<cuuint64_t>(P)};
        const cuuint64_t str[2] = {static_cast<cuuint64_t>(8 * ldm), static_cast<cuuint64_t>(8 * e_stride)};
        const cuuint32_t box[3] = {8, 16, 1};
        if (enc(&M.x, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(earlier), dims, str, box, e1,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return pint_set_error(ctx, PINT_E_CUDA, "affine_pair: tensor map x failed");
    }
    pint_kernel_attrs(reinterpret_cast<const void*>(affine_pair_tma_kernel));
    const long long t = (n + 127) / 128, tiles = P * t * t;
    // Persistent, one CTA per SM, each taking a CONTIGUOUS run of tiles (the next tile's first k
    // tiles load during this one's epilogue). Measured at n = 512, 128 pairs: 31.7 TFLOP/s, against
    // 29.8 for one tile per CTA and 27.0 for the same persistent grid with tiles dealt round-robin
    // (cuBLAS batched DGEMM: 30.9). PINT_PAIR_GRID / PINT_PAIR_CHUNK=0: experiments.
    static const long long grid_env = [] {
        const char* e = std::getenv("PINT_PAIR_GRID");
        return e ? std::atoll(e) : 0ll;
    }();
    const unsigned grid = static_cast<unsigned>(std::min<long long>(tiles, grid_env ? grid_env : ctx->sm_count));
    static const int chunk_env = [] {
        const char* e = std::getenv("PINT_PAIR_CHUNK");
        return e ? std::atoi(e) : 1;
    }();
    affine_pair_tma_kernel<<<grid, 256, pair_tma_smem(), ctx->stream>>>(M, static_cast<int>(n), ldm,
                                                                        static_cast<int>(P), later, l_stride, out,
                                                                        o_stride, chunk_env);
    return pint_check_launch(ctx, "affine_pair_tma_kernel");
}

template <int MI>
int launch_pairs_mi(pint_ctx* ctx, long long n, long long P, const double* earlier, long long e_stride,
                    const double* later, long long l_stride, double* out, long long o_stride) {
    const long long ldm = pint_affine_ldm(n);
    const unsigned tilesN = static_cast<unsigned>((n + BN - 1) / BN);  // (column n: see affine_pair_kernel)
    const unsigned tilesM = static_cast<unsigned>((n + 16 * MI - 1) / (16 * MI));
    dim3 grid(tilesN, tilesM, static_cast<unsigned>(P));
    constexpr size_t smem = pair_smem_bytes<MI>();
    static bool attr = [] {
        return cudaFuncSetAttribute(affine_pair_kernel<MI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)) == cudaSuccess;
    }();
    (void)attr;
    affine_pair_kernel<MI><<<grid, 128, smem, ctx->stream>>>(n, ldm, earlier, e_stride, later, l_stride, out,
                                                             o_stride);
    return pint_check_launch(ctx, "affine_pair_kernel");
}

int launch_pairs(pint_ctx* ctx, long long n, long long P, const double* earlier, long long e_stride,
                 const double* later, long long l_stride, double* out, long long o_stride) {
    if (P <= 0) return PINT_OK;
    if (P > 65535) return pint_set_error(ctx, PINT_E_INVALID, "affine_pair: too many pairs per launch");
    // PINT_PAIR_MI: tile-shape experiments only
    static const int mi_env = [] {
        const char* e = std::getenv("PINT_PAIR_MI");
        return e ? std::atoi(e) : 0;
    }();
    // 128-row tiles (warp tile 64 x 32: half the B-fragment loads per DMMA) pay once the grid is
    // large enough to fill the SMs anyway (n = 512: tree -9%); at n = 128 the 64-row tiles win
    // the TMA-fed 128 x 128 kernel where 16 | n (PINT_PAIR_TMA=0: the cp.async kernel)
    static const int tma_env = [] {
        const char* e = std::getenv("PINT_PAIR_TMA");
        return e ? std::atoi(e) : 1;
    }();
    // Measured (tools/prof_pair.py, n = 512): the TMA kernel from 8 pairs up (29.8-30.7 TFLOP/s at
    // 128 pairs, cuBLAS batched DGEMM 30.9), the 128 x 64 cp.async tiles otherwise, and 64 x 64 tiles
    // when even those leave SMs idle (2-4 pairs: 11.7-17.2 against 7.3-14.1). Where 128 does not
    // divide n the 128-wide TMA tiles waste work (n = 144: 5.9 against 8.0); below n = 384 the
    // cp.async kernel is as fast.
    const long long t128 = n / 128;
    if (tma_env && !mi_env && n % 128 == 0 && n >= 384 && 2 * P * t128 * t128 >= ctx->sm_count)
        return launch_pairs_tma(ctx, n, P, earlier, e_stride, later, l_stride, out, o_stride);
    int mi = mi_env ? mi_env : n >= 384 ? 8 : 4;
    if (!mi_env && mi == 8 && P * ((n + 127) / 128) * ((n + BN - 1) / BN) < ctx->sm_count) mi = 4;
    if (mi == 8) return launch_pairs_mi<8>(ctx, n, P, earlier, e_stride, later, l_stride, out, o_stride);
    if (mi == 6) return launch_pairs_mi<6>(ctx, n, P, earlier, e_stride, later, l_stride, out, o_stride);
    return launch_pairs_mi<4>(ctx, n, P, earlier, e_stride, later, l_stride, out, o_stride);
}

}  // namespace

int launch_affine_chain(pint_ctx* ctx, int64_t n, int64_t N, const double* maps, const double* y0,
                        double* y) {
    return launch_affine_chain_on(ctx, ctx->stream, n, N, maps, y0, y, nullptr, 0);
}

int launch_affine_chain_on(pint_ctx* ctx, cudaStream_t stream, int64_t n, int64_t N, const double* maps,
                           const double* y0, double* y, const int* ready, int target, int wide_chain_rows) {
    if (n < 1 || N < 0) return pint_set_error(ctx, PINT_E_INVALID, "affine_chain: bad sizes");
    // the wide chain (TMA-streamed, 32 W rows per CTA) for 256 < n <= 512 with n % 16 == 0: W = 4
    // beside the exact build (wide_rows 128: it keeps up with the build on 4 SMs, the build gets
    // 144), else W = 2 (the fastest shape: 3.6 us per map at n = 512 on 8 SMs, against 4.8 us for the
    // 16-CTA cluster chain). PINT_WIDE_CHAIN=0 turns it off, PINT_WIDE_W forces W (experiments).
    static const int wide_env = [] {
        const char* e = std::getenv("PINT_WIDE_CHAIN");
        return e ? std::atoi(e) : 1;
    }();
    static const int wide_w = [] {
        const char* e = std::getenv("PINT_WIDE_W");
        const int w = e ? std::atoi(e) : 0;
        return w == 1 || w == 2 || w == 4 ? w : 0;
    }();
    const int W = wide_w ? wide_w : (ready && wide_chain_rows >= 128) ? 4 : 2;
    if (wide_env && n > 256 && n <= 512 && n % 16 == 0 && N > 0 && (n + 32 * W - 1) / (32 * W) <= 16) {
        const int ldm = static_cast<int>(pint_affine_ldm(n));
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(pint_tensor_map_encoder());
        if (!enc) return pint_set_error(ctx, PINT_E_CUDA, "affine_chain: cuTensorMapEncodeTiled unavailable");
        CUtensorMap tm;
        const cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(n / 16),
                                    static_cast<cuuint64_t>(N)};
        const cuuint64_t strides[3] = {static_cast<cuuint64_t>(8 * ldm), 128,
                                       static_cast<cuuint64_t>(8 * static_cast<int64_t>(n) * ldm)};
        const cuuint32_t box[4] = {16, 32, kWideBlk, 1}, estr[4] = {1, 1, 1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(maps), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return pint_set_error(ctx, PINT_E_CUDA, "affine_chain: tensor map failed");
        const size_t ny = static_cast<size_t>((n + kWideCols - 1) / kWideCols * kWideCols);
        const size_t smem = 1024 + sizeof(double) * (kWideRingTotal * kWideSlot + 2 * ny) + 8 * (2 * kWideRingTotal + 2);
        auto kern = W == 4 ? affine_chain_wide_kernel<4> : W == 2 ? affine_chain_wide_kernel<2> : affine_chain_wide_kernel<1>;
        pint_kernel_attrs(reinterpret_cast<const void*>(kern));
        const unsigned C = static_cast<unsigned>((n + 32 * W - 1) / (32 * W));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C, 1, 1);
        cfg.blockDim = dim3(32 * (W + 1), 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, tm, static_cast<int>(n), static_cast<long long>(N), ldm, maps, y0, y, ready,
                           target, ctx->d_fail);
        return pint_check_launch(ctx, "affine_chain_wide_kernel");
    }
    if (n <= 32 * kClusterMax && N > 0) {
        const int ldm = static_cast<int>(pint_affine_ldm(n));
        const size_t ny = static_cast<size_t>((n + 15) & ~15);
        const size_t blk = sizeof(double) * 32 * static_cast<size_t>(ldm);
        const size_t rest = sizeof(double) * (2 * ny + 4 * kChainAhead) + 8 * (kRing + 2);
        const int ring = static_cast<int>(std::min<size_t>(kRing, (227 * 1024 - rest) / blk));
        const size_t smem = ring * blk + rest;
        pint_kernel_attrs(reinterpret_cast<const void*>(affine_chain_cluster_kernel));
        const unsigned C = static_cast<unsigned>((n + 31) / 32);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C, 1, 1);
        cfg.blockDim = dim3(32, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, affine_chain_cluster_kernel, static_cast<int>(n), static_cast<long long>(N), ldm,
                               ring, maps, y0, y, ready, target, ctx->d_fail) != cudaSuccess)
            return pint_check_launch(ctx, "affine_chain_cluster_kernel");
        return pint_check_launch(ctx, "affine_chain_cluster_kernel");
    }
    if (n > 4 * kChainThreads) return pint_set_error(ctx, PINT_E_INVALID, "affine_chain: n > 1024 unsupported");
    if (ready) return pint_set_error(ctx, PINT_E_INVALID, "affine_chain: waiting on builders needs n <= 512");
    const size_t smem = sizeof(double) * static_cast<size_t>(n);
    affine_chain_kernel<<<1, kChainThreads, smem, stream>>>(n, N, pint_affine_ldm(n), maps, y0, y);
    return pint_check_launch(ctx, "affine_chain_kernel");
}

int launch_affine_pair(pint_ctx* ctx, int64_t n, int64_t P, const double* earlier,
                       const double* later, double* out) {
    const long long stride = n * pint_affine_ldm(n);
    return launch_pairs(ctx, n, P, earlier, stride, later, stride, out, stride);
}

// The log-depth tree: level by level, pairs (2p, 2p+1) of `src` into `dst`, odd tail copied.
// Maps left for the chain when only y is wanted: a pair level costs >= ~14 us even for a handful
// of GEMMs, the cluster chain ~1.5 us per map (n = 128), so the last 4 levels become a chain.
constexpr long long kTreeChainTail = 16;

int launch_affine_tree(pint_ctx* ctx, int64_t n, int64_t N, double* maps, double* scratch,
                       const double* y0, double* y, double* composed) {
    if (N < 1) return pint_set_error(ctx, PINT_E_INVALID, "affine_tree: N >= 1 required");
    const long long stride = n * pint_affine_ldm(n);
    double* src = maps;
    double* dst = scratch;
    long long count = N;
    // When only y is wanted, pairing may stop once a level would be latency-bound (a pair level
    // costs ~14 us even for a handful of GEMMs) and the chain applies the rest. Past n = 256 the
    // chain (a 16-CTA cluster at n = 512: ~5.3 us per map) is cheaper per map than the products
    // (2 n^3 flops: ~10 us a map at n = 512 on the DMMA pipe), so there only-y skips the tree
    // entirely — and the result is the bit-exact chain's.
    const long long stop = composed ? 1 : n > 256 ? N : kTreeChainTail;
    while (count > stop) {
        const long long pairs = count / 2;
        for (long long p0 = 0; p0 < pairs; p0 += 65535) {
            const long long P = (pairs - p0 < 65535) ? pairs - p0 : 65535;
            const int rc = launch_pairs(ctx, n, P, src + 2 * p0 * stride, 2 * stride,
                                        src + (2 * p0 + 1) * stride, 2 * stride, dst + p0 * stride, stride);
            if (rc) return rc;
        }
        if (count & 1) {
            if (cudaMemcpyAsync(dst + pairs * stride, src + (count - 1) * stride, sizeof(double) * stride,
                                cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
                return pint_set_error(ctx, PINT_E_CUDA, "affine_tree: tail copy failed");
        }
        double* t = src;
        src = dst;
        dst = t;
        count = pairs + (count & 1);
    }
    if (composed && composed != src &&
        cudaMemcpyAsync(composed, src, sizeof(double) * stride, cudaMemcpyDeviceToDevice, ctx->stream) != cudaSuccess)
        return pint_set_error(ctx, PINT_E_CUDA, "affine_tree: composed copy failed");
    return launch_affine_chain(ctx, n, count, src, y0, y);
}
