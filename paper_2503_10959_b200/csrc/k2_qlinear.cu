// K2 — mixed-precision quant-linear: int8/int4-code inlier GEMM on the 5th-gen
// tensor cores (tcgen05.mma kind::i8, int32 accumulators in TMEM) with the
// hybrid epilogue of the reference fused in (gemm.cpp:181-225):
//
//   acc[m][r]  = sum_k x_code[m][k] * w_code[r][k]            (exact int32)
//   y          = S_m * acc                                    gemm.cpp:207
//   y         += (s_j * w[r][ch_j]) * xo_j   for j ascending   gemm.cpp:208-216
//   y          = ws[r] * y                                    gemm.cpp:218-219
//
// then the layer's post-op (in_proj split + SiLU gate, D1 residual add, ...).
// Orientation: the reference computes y[out][token] with activations K x C;
// here rows are tokens (A = activation codes, M x K, K-major) and columns are
// output features (B = weight codes, R x K, K-major), so both operands are the
// canonical K-major UMMA layout and the output rows are the next layer's
// token-major activations.
//
// Structure (persistent, one CTA per SM; 4 + EW warps, EW = 8 or 16 epilogue warps):
//   warp 0      TMA producer: 128x128 A tile + BNx128 B tile per K-block, 128B swizzle
//   warp 1      MMA issuer: 4 x tcgen05.mma.kind::i8 (M=128, N=BN, K=32) per K-block
//   warp 2      TMEM allocator (2 x BN columns: double-buffered accumulators)
//   warp 3      row metadata (S_m, |O(t)|, mask words) of upcoming tiles, bulk-copied
//   warps 4..   epilogue: tcgen05.ld 32x32b, f64 dequant + outlier terms per row, then
//               ws[r] * y, the post-op and TMA stores of 32x16 f64 boxes from swizzled staging
//   last 4      (A4 nibble-packed activations, PK) unpack warpgroup: the producer's TMA puts
//               the stage's packed 128 x 64-byte A box into the upper half of the stage's A
//               region; these warps expand it in place to the 128B-swizzled int8 tile
//               (pack_int4's layout, gemm.cpp:60-73: low nibble = even channel), fence it to
//               the async proxy and arrive on the stage's full barrier next to the TMA bytes
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"
#include "sm100_ptx.cuh"

namespace ob {

constexpr int kBM = 128, kBK = 128;
constexpr int kStgBufs = 1;  // epilogue staging buffers per warp
// Shapes of the same kernel, chosen per call (launch_qlinear). The f64 epilogue, not the
// int8 main loop, bounds K2 (Vim-B in_proj: main loop alone 61 of 159 us; each epilogue
// warp's chunks are a serial chain of TMEM load, f64 dequant / outlier terms, staging and
// the TMA store's smem read), so more epilogue warps pay where the grid is full:
//  * ONEBOX: 16 epilogue warps (setmaxnreg moving registers from warpgroup 0), one 4 KB
//    staging box per warp reused by the chunk's two boxes, 4 operand stages — calls of at
//    least a wave of tiles, K <= 1024, no residual (in_proj 141 vs 159 us, x_proj 87 vs
//    95 us with the 8-warp shape);
//  * 16 epilogue warps, two boxes per warp, 2 stages: the residual post-op (its tile is
//    loaded into the boxes) and narrow calls below a wave;
//  * 8 epilogue warps, 4 stages: wide calls below a wave or with K > 1024 (its hoisted,
//    vectorised outlier walk); with the unpack warpgroup for the packed A4 operand (PK).
template <int EW, bool PK = false>
struct K2Cfg {
    static constexpr int kEpiWarps = EW;
    static constexpr int kUnpackWarps = PK ? 4 : 0;
    static constexpr int kThreads = 128 + 32 * EW + 32 * kUnpackWarps;
    static constexpr int kStages = EW >= 16 ? 2 : 4;
    static constexpr int kMaskWords = 24;  // mask words per row staged in shared memory (K <= 768; else global)
};

// ONEBOX (16 epilogue warps, no residual): one 4 KB staging box per warp, reused by the
// chunk's two boxes, pays for four operand stages instead of two (16 x 4 KB + 4 x 32 KB +
// metadata = 225 KB)
template <int BN, int EW, bool ONEBOX = false>
struct K2Smem {
    static constexpr int kStages = ONEBOX ? 4 : K2Cfg<EW>::kStages, kEpiWarps = EW, kMaskWords = K2Cfg<EW>::kMaskWords;
    static constexpr int kStgBytes = ONEBOX ? 4096 : 8192;
    static constexpr int kABytes = kBM * kBK;
    static constexpr int kBBytes = BN * kBK;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kEpiOff = kStages * kStageBytes;  // per warp: 2 x (32 x 32 f64 output tile = 2 TMA boxes)
    static constexpr int kWsOff = kEpiOff + kEpiWarps * kStgBufs * kStgBytes;  // per warp: the chunk's 32 column scales
    // row metadata ring (2 tiles ahead, filled by warp 3): S_m, |O|, mask words (J <= 32)
    static constexpr int kMetaS = 0, kMetaCnt = kBM * 8, kMetaMask = kMetaCnt + kBM * 4;
    static constexpr int kMetaBytes = kMetaMask + kBM * kMaskWords * 4;
    static constexpr int kMetaOff = kWsOff + kEpiWarps * 256;
    static constexpr int kBarOff = kMetaOff + 2 * kMetaBytes;
    static constexpr int kTotal = kBarOff + 512 + 1024;  // barriers + tmem slot + alignment slack
};

// Eight pack_int4 codes (one 32-bit word, low nibble = even channel) -> eight int8
// codes in channel order: each nibble sign-extended into its byte ((n & 8) * 0x1E puts
// 0xF0 over a negative nibble; no carries cross bytes), then the even / odd bytes
// interleaved.
__device__ __forceinline__ void unpack_nibbles8(uint32_t x, uint32_t& o0, uint32_t& o1) {
    const uint32_t lo = x & 0x0F0F0F0Fu, hi = (x >> 4) & 0x0F0F0F0Fu;
    const uint32_t rlo = (lo & 0x08080808u) * 0x1Eu + lo, rhi = (hi & 0x08080808u) * 0x1Eu + hi;
    o0 = __byte_perm(rlo, rhi, 0x5140);
    o1 = __byte_perm(rlo, rhi, 0x7362);
}

// 32 packed codes (16 bytes) of row r, channel quarter kq of the K-block -> the two
// 16-byte chunks 2kq, 2kq+1 of the 128B-swizzled int8 row
__device__ __forceinline__ void unpack_chunk(uint8_t* sa, int r, int kq, uint4 x) {
    uint4 a, b;
    unpack_nibbles8(x.x, a.x, a.y);
    unpack_nibbles8(x.y, a.z, a.w);
    unpack_nibbles8(x.z, b.x, b.y);
    unpack_nibbles8(x.w, b.z, b.w);
    uint8_t* row = sa + r * 128;
    *reinterpret_cast<uint4*>(row + (((2 * kq) ^ (r & 7)) << 4)) = a;
    *reinterpret_cast<uint4*>(row + (((2 * kq + 1) ^ (r & 7)) << 4)) = b;
}

// int32 -> f64, exact, without the conversion pipe (I2F.F64 is slow on sm_100):
// 2^52 + (v + 2^31) assembled from words, minus 2^52 + 2^31.
__device__ __forceinline__ double i32_to_f64(uint32_t v) {
    return __hiloint2double(0x43300000, static_cast<int>(v ^ 0x80000000u)) - 4503601774854144.0;
}

template <int BN, int EW, int POST, bool PLANES, bool PK, bool ONEBOX>
__global__ void __launch_bounds__(K2Cfg<EW, PK>::kThreads, 1)
    k2_qlinear(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO2, const QLinParams p) {
    static_assert(!ONEBOX || (EW >= 16 && POST != POST_RESID && !PK), "one-box staging: 16 warps, no residual");
    using L = K2Smem<BN, EW, ONEBOX>;
    constexpr int kStages = L::kStages, kEpiWarps = EW, kMaskWords = L::kMaskWords;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned for the 128B-swizzled tiles; indexed from the shared array (no integer
    // round trip) so the compiler keeps the shared window: LDS / STS, not generic LD / ST
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* empty = full + kStages;
    uint64_t* acc_full = empty + kStages;
    uint64_t* acc_empty = acc_full + 2;
    uint64_t* res_bar = acc_empty + 2;  // per epilogue warp and staging buffer: residual tile loads
    uint64_t* meta_full = res_bar + 2 * kEpiWarps;
    uint64_t* meta_empty = meta_full + 2;
    uint64_t* pk_full = meta_empty + 2;  // PK: the stage's packed A box landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pk_full + kStages);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m_tiles = (p.M + kBM - 1) / kBM, n_tiles = (p.R + BN - 1) / BN;
    const int tiles = m_tiles * n_tiles;
    const int kblocks = (p.K + kBK - 1) / kBK;

    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(full + s, PK ? 1 + 4 : 1);  // PK: + one arrive per unpack warp
            ptx::mbar_init(empty + s, 1);
            ptx::mbar_init(pk_full + s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(acc_full + s, 1);
            ptx::mbar_init(acc_empty + s, kEpiWarps);  // one arrive per epilogue warp
        }
        for (int w = 0; w < 2 * kEpiWarps; ++w) ptx::mbar_init(res_bar + w, 1);
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(meta_full + s, 1);
            ptx::mbar_init(meta_empty + s, kEpiWarps);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<2 * BN>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // warpgroup 0 (TMA, MMA, TMEM allocator, row metadata) needs few registers: it hands
    // them to the four epilogue warpgroups (register budgets per role region)
    // (PK adds a warpgroup: the 8-epilogue-warp shape then moves registers too)
    constexpr bool kRegMove = EW >= 16 || PK;
    if (warp < 4) {
    if constexpr (kRegMove) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
                const int m0 = (tile / n_tiles) * kBM, n0 = (tile % n_tiles) * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    ptx::mbar_wait(empty + stage, phase ^ 1);
                    uint8_t* sa = smem + stage * L::kStageBytes;
                    if constexpr (PK) {  // packed A box (128 rows x 64 bytes) into the A region's upper half
                        ptx::mbar_arrive_expect_tx(pk_full + stage, L::kABytes / 2);
                        ptx::tma_load_2d(sa + L::kABytes / 2, &tmA, pk_full + stage, kb * (kBK / 2), m0);
                        ptx::mbar_arrive_expect_tx(full + stage, L::kBBytes);
                    } else {
                        ptx::mbar_arrive_expect_tx(full + stage, L::kStageBytes);
                        ptx::tma_load_2d(sa, &tmA, full + stage, kb * kBK, m0);
                    }
                    ptx::tma_load_2d(sa + L::kABytes, &tmB, full + stage, kb * kBK, n0);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc = ptx::idesc_i8(kBM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
                const int buf = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ptx::mbar_wait(acc_empty + buf, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + buf * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    ptx::mbar_wait(full + stage, phase);
                    ptx::tc_fence_after();
                    uint8_t* sa = smem + stage * L::kStageBytes;
                    const uint64_t da = ptx::smem_desc_sw128(sa);
                    const uint64_t db = ptx::smem_desc_sw128(sa + L::kABytes);
#pragma unroll
                    for (int k = 0; k < kBK / 32; ++k)  // K=32 bytes per MMA: +2 in 16-byte units
                        ptx::mma_i8(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                    ptx::mma_commit(empty + stage);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit(acc_full + buf);
            }
        }
    } else if (warp == 3) {  // ---- row metadata producer: S_m, |O| and mask words of upcoming tiles
        const int J = p.a.J;
        const bool smask = J <= kMaskWords;  // mask rows fit the slot; else the epilogue reads them globally
        const bool bulk_ok = ((reinterpret_cast<uintptr_t>(p.a.s_row) | reinterpret_cast<uintptr_t>(p.a.ocnt) |
                               reinterpret_cast<uintptr_t>(p.a.omask)) & 15) == 0;
        int it = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
            const int slot = it & 1;
            ptx::mbar_wait(meta_empty + slot, ((it >> 1) & 1) ^ 1);
            uint8_t* mb = smem + L::kMetaOff + slot * L::kMetaBytes;
            double* ms = reinterpret_cast<double*>(mb + L::kMetaS);
            int* mc = reinterpret_cast<int*>(mb + L::kMetaCnt);
            uint32_t* mm = reinterpret_cast<uint32_t*>(mb + L::kMetaMask);
            const int m0 = (tile / n_tiles) * kBM;
            const int nrows = min(kBM, p.M - m0);
            if (nrows == kBM && bulk_ok) {  // full tile: three contiguous bulk copies onto the slot's barrier
                if (lane == 0) {
                    const uint32_t mbytes = smask ? static_cast<uint32_t>(kBM * J * 4) : 0u;
                    ptx::mbar_arrive_expect_tx(meta_full + slot, kBM * 8 + kBM * 4 + mbytes);
                    ptx::bulk_g2s(ms, p.a.s_row + m0, kBM * 8, meta_full + slot);
                    ptx::bulk_g2s(mc, p.a.ocnt + m0, kBM * 4, meta_full + slot);
                    if (smask) ptx::bulk_g2s(mm, p.a.omask + static_cast<size_t>(m0) * J, mbytes, meta_full + slot);
                }
                continue;
            }
#pragma unroll
            for (int i = lane; i < kBM; i += 32) {  // ragged last tile
                const bool v = i < nrows;
                ms[i] = v ? __ldg(p.a.s_row + m0 + i) : 0.0;
                mc[i] = v ? __ldg(p.a.ocnt + m0 + i) : 0;
            }
            if (smask) {
                const uint32_t* src = p.a.omask + static_cast<size_t>(m0) * J;
                const int n = nrows * J;
                for (int i = lane; i < n; i += 32) mm[i] = __ldg(src + i);
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(meta_full + slot);
        }
    }
    } else if (PK && warp >= 4 + EW) {  // ---- unpack warpgroup (PK)
        static_assert(!PK || EW == 8, "the unpack warpgroup's register budget is laid out for 8 epilogue warps");
        if constexpr (kRegMove) asm volatile("setmaxnreg.dec.sync.aligned.u32 48;\n" ::: "memory");
        const int u = threadIdx.x - 32 * (4 + EW);  // 0..127
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            for (int kb = 0; kb < kblocks; ++kb) {
                uint8_t* sa = smem + stage * L::kStageBytes;
                const uint8_t* pk = sa + L::kABytes / 2;  // packed row r at pk + 64 r
                ptx::mbar_wait(pk_full + stage, phase);
                // in place: rows 0..63 expand into [0, 8 KB), below the packed box; rows
                // 64..127 expand over it, so their packed bytes are read first and every
                // read of the group precedes the second half's writes (named barrier)
                const uint4 h0 = *reinterpret_cast<const uint4*>(pk + 4096 + u * 16);
                const uint4 h1 = *reinterpret_cast<const uint4*>(pk + 4096 + (u + 128) * 16);
#pragma unroll
                for (int i = u; i < 256; i += 128) unpack_chunk(sa, i >> 2, i & 3, *reinterpret_cast<const uint4*>(pk + i * 16));
                asm volatile("bar.sync 1, 128;" ::: "memory");
                unpack_chunk(sa, 64 + (u >> 2), u & 3, h0);
                unpack_chunk(sa, 64 + ((u + 128) >> 2), u & 3, h1);
                ptx::fence_async_smem();  // generic-proxy writes -> the tensor core's async proxy
                __syncwarp();
                if ((u & 31) == 0) ptx::mbar_arrive(full + stage);
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else {  // ---- epilogue: 16 warps = 4 TMEM lane quarters x 4 column groups
        // register budgets within the CTA's pool (threads x launch registers): 128 x 40 (+ 128 x 48
        // unpack) + 32 EW x epilogue, i.e. 640 x 96 >= 128 x 40 + 512 x 104 and 512 x 128 >=
        // 128 x 40 + 128 x 48 + 256 x 200
        if constexpr (EW >= 16) asm volatile("setmaxnreg.inc.sync.aligned.u32 104;\n" ::: "memory");
        else if constexpr (PK) asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
        const int ew = warp - 4;
        const int q = warp & 3;       // TMEM lanes 32q..32q+31 (a warp may only touch its quarter)
        const int cgrp = ew >> 2;     // which quarter of the BN columns
        // per-warp output tiles (double-buffered): two 32-row x 16-double boxes each, 128B-swizzled
        uint8_t* stg0 = smem + L::kEpiOff + ew * kStgBufs * L::kStgBytes;
        constexpr bool kOneBox = L::kStgBytes == 4096;  // the chunk's two boxes pass through one buffer
        double* wss = reinterpret_cast<double*>(smem + L::kWsOff + ew * 256);

        constexpr bool resid = POST == POST_RESID;
        int it = 0, cs = 0;  // tile and chunk sequence of this warp
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
            const int buf = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            const int m0 = (tile / n_tiles) * kBM, n0 = (tile % n_tiles) * BN;
            const int rbase = m0 + q * 32;
            const int row = rbase + lane;
            const bool rv = row < p.M;
            const int mslot = it & 1;
            ptx::mbar_wait(meta_full + mslot, (it >> 1) & 1);
            const uint8_t* mb = smem + L::kMetaOff + mslot * L::kMetaBytes;
            const double S = reinterpret_cast<const double*>(mb + L::kMetaS)[q * 32 + lane];
            const int cnt = reinterpret_cast<const int*>(mb + L::kMetaCnt)[q * 32 + lane];
            const uint32_t* msk = p.a.J <= kMaskWords
                                      ? reinterpret_cast<const uint32_t*>(mb + L::kMetaMask) + (q * 32) * p.a.J
                                              : p.a.omask + static_cast<size_t>(rbase) * p.a.J;
            // the row's outlier channels, codes and scales are the same for every column chunk
            // of the tile: fetched once (up to kHoist), before the accumulator wait hides their
            // latency
            // (8-epilogue-warp shape only: the 16-warp shape's register budget would spill)
            constexpr int kHoist = EW >= 16 ? 1 : 4;
            int hch[kHoist], hxo[kHoist];
            double hosc[kHoist];
            const bool hoisted = EW < 16 && cnt <= kHoist;
            if (cnt > 0 && hoisted) {
                int word = -1;
                unsigned bits = 0;
#pragma unroll
                for (int o = 0; o < kHoist; ++o) {
                    if (o < cnt) {
                        while (bits == 0) bits = msk[lane * p.a.J + (++word)];
                        hch[o] = word * 32 + (__ffs(bits) - 1);
                        bits &= bits - 1;
                        const size_t oi = static_cast<size_t>(row) * p.K + hch[o];
                        hxo[o] = p.a.ocode[oi];
                        hosc[o] = p.a.oscale[oi];
                    }
                }
            }
            constexpr int kChunksPerWarp = BN / 32 / (EW / 4);
            // column scales ws[r] of the warp's first chunk, loaded before the accumulator wait;
            // each chunk prefetches the next one's (an L2 round trip per chunk otherwise)
            const int rfirst = n0 + cgrp * kChunksPerWarp * 32;
            double wsn = rfirst < p.R ? __ldg(p.ws + rfirst + lane) : 0.0;
            // the first outlier channel's 32 weights of the warp's first chunk, loaded before the
            // accumulator wait; each chunk prefetches the next chunk's (8-warp shape)
            int4 pw0 = make_int4(0, 0, 0, 0), pw1 = make_int4(0, 0, 0, 0);
            const bool pre0 = EW < 16 && hoisted && cnt > 0;
            if (pre0 && rfirst < p.R) {
                const int4* wp = reinterpret_cast<const int4*>(p.wt + static_cast<size_t>(hch[0]) * p.R + rfirst);
                pw0 = __ldg(wp);
                pw1 = __ldg(wp + 1);
            }
            ptx::mbar_wait(acc_full + buf, aphase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int cc = 0; cc < kChunksPerWarp; ++cc, ++cs) {
                const int c = cgrp * kChunksPerWarp + cc;
                const int r0 = n0 + c * 32;
                if (r0 >= p.R) break;  // uniform across the warp
                const double wsl = wsn;  // R % 32 == 0: in range
                if (cc + 1 < kChunksPerWarp && r0 + 32 < p.R) wsn = __ldg(p.ws + r0 + 32 + lane);
                const bool to2 = POST == POST_INPROJ && r0 >= p.epi.split;
                const CUtensorMap* om = to2 ? &tmO2 : &tmO;
                const int oc0 = to2 ? r0 - p.epi.split : r0;
                const int sb = kStgBufs == 2 ? (cs & 1) : 0;
                uint8_t* stg = stg0 + sb * L::kStgBytes;
                uint64_t* rbar = res_bar + 2 * ew + sb;
                if (lane == 0) {
                    if (kStgBufs == 2) ptx::bulk_wait_read1();  // this buffer's store (two chunks ago) has left it
                    else ptx::bulk_wait_read0();
                    if (resid) {             // D1 residual: bring x[rows][r0..r0+31] into the staging tile
                        ptx::mbar_arrive_expect_tx(rbar, 8192);
                        ptx::tma_load_2d(stg, om, rbar, oc0, rbase);
                        ptx::tma_load_2d(stg + 4096, om, rbar, oc0 + 16, rbase);
                    }
                }
                __syncwarp();
                uint32_t acc[32];
                ptx::tmem_ld32(tmem_base + ((q * 32) << 16) + buf * BN + c * 32, acc);
                // thread = row: S_m * acc (gemm.cpp:207), outlier terms in ascending channel
                // order (gemm.cpp:208-216), ws[r] * y (gemm.cpp:218-219), post-op
                double y[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) y[j] = dmul(S, i32_to_f64(acc[j]));
                int32_t aout[PLANES ? 32 : 1];
                if (PLANES)
#pragma unroll
                    for (int j = 0; j < 32; ++j) aout[j] = 0;
                // outlier terms in ascending channel order (gemm.cpp:208-216)
                auto outlier_term_w = [&](int xo_i, double osc, int4 w01, int4 w23) {
                    const double xo = i32_to_f64(static_cast<uint32_t>(xo_i));
                    const int wd[8] = {w01.x, w01.y, w01.z, w01.w, w23.x, w23.y, w23.z, w23.w};
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int wq = static_cast<int8_t>(static_cast<uint32_t>(wd[j >> 2]) >> (8 * (j & 3)));  // register byte
                        const double coeff = dmul(osc, i32_to_f64(static_cast<uint32_t>(wq)));
                        y[j] = dadd(y[j], dmul(coeff, xo));
                        if (PLANES) aout[j] += wq * xo_i;
                    }
                };
                auto outlier_term = [&](int ch, int xo_i, double osc) {
                    const int4* wp = reinterpret_cast<const int4*>(p.wt + static_cast<size_t>(ch) * p.R + r0);
                    outlier_term_w(xo_i, osc, __ldg(wp), __ldg(wp + 1));
                };
                if (hoisted) {
                    if (pre0) {  // the prefetched weights of channel hch[0]; the next chunk's in flight
                        const int4 w01 = pw0, w23 = pw1;
                        if (cc + 1 < kChunksPerWarp && r0 + 32 < p.R) {
                            const int4* wp = reinterpret_cast<const int4*>(p.wt + static_cast<size_t>(hch[0]) * p.R + r0 + 32);
                            pw0 = __ldg(wp);
                            pw1 = __ldg(wp + 1);
                        }
                        outlier_term_w(hxo[0], hosc[0], w01, w23);
                    }
#pragma unroll
                    for (int o = 0; o < kHoist; ++o)
                        if (o < cnt && !(o == 0 && pre0)) outlier_term(hch[o], hxo[o], hosc[o]);
                } else if (EW >= 16) {  // more than kHoist (16-warp shape: its register budget): word by word
                    int word = -1;
                    unsigned bits = 0;
                    for (int o = 0; o < cnt; ++o) {
                        while (bits == 0) bits = msk[lane * p.a.J + (++word)];
                        const int ch = word * 32 + (__ffs(bits) - 1);
                        bits &= bits - 1;
                        const size_t oi = static_cast<size_t>(row) * p.K + ch;
                        outlier_term(ch, p.a.ocode[oi], p.a.oscale[oi]);
                    }
                } else {  // more than kHoist: the mask walked 4 words per load (J % 4 == 0), the next
                          // outlier's code, scale and weights in flight while this one's terms run
                    const uint32_t* mrow = msk + lane * p.a.J;
                    const bool vec = (p.a.J & 3) == 0;
                    int word = 0, gi = 4, wbase = 0;
                    uint4 grp = make_uint4(0u, 0u, 0u, 0u);
                    unsigned bits = 0;
                    auto next_ch = [&]() {
                        while (bits == 0) {
                            if (vec) {
                                if (gi == 4) {
                                    grp = *reinterpret_cast<const uint4*>(mrow + word);
                                    word += 4;
                                    gi = 0;
                                }
                                bits = gi == 0 ? grp.x : (gi == 1 ? grp.y : (gi == 2 ? grp.z : grp.w));
                                wbase = (word - 4 + gi) * 32;
                                ++gi;
                            } else {
                                bits = mrow[word];
                                wbase = word * 32;
                                ++word;
                            }
                        }
                        const int ch = wbase + __ffs(bits) - 1;
                        bits &= bits - 1;
                        return ch;
                    };
                    int xo = 0;
                    double osc = 0.0;
                    int4 wa = make_int4(0, 0, 0, 0), wb = make_int4(0, 0, 0, 0);
                    auto fetch = [&]() {
                        const int ch = next_ch();
                        const size_t oi = static_cast<size_t>(row) * p.K + ch;
                        xo = p.a.ocode[oi];
                        osc = p.a.oscale[oi];
                        const int4* wp = reinterpret_cast<const int4*>(p.wt + static_cast<size_t>(ch) * p.R + r0);
                        wa = __ldg(wp);
                        wb = __ldg(wp + 1);
                    };
                    if (cnt > 0) fetch();
                    for (int o = 0; o < cnt; ++o) {
                        const int xo_c = xo;
                        const double osc_c = osc;
                        const int4 wa_c = wa, wb_c = wb;
                        if (o + 1 < cnt) fetch();
                        outlier_term_w(xo_c, osc_c, wa_c, wb_c);
                    }
                }
                if (PLANES && rv) {  // the reference's integer planes (parity path)
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        p.epi.acc_in[static_cast<size_t>(row) * p.R + r0 + j] = static_cast<int32_t>(acc[j]);
                        p.epi.acc_out[static_cast<size_t>(row) * p.R + r0 + j] = aout[j];
                    }
                }
                wss[lane] = wsl;
                __syncwarp();
                if (resid) ptx::mbar_wait(rbar, (kStgBufs == 2 ? cs >> 1 : cs) & 1);
#pragma unroll
                for (int j2 = 0; j2 < 16; ++j2) {  // 16-byte chunk j2 = columns 2*j2, 2*j2+1
                    if (kOneBox && j2 == 8) {  // box 0 leaves, then box 1 reuses the buffer
                        ptx::fence_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_2d(om, stg, oc0, rbase);
                            ptx::bulk_commit();
                            ptx::bulk_wait_read0();
                        }
                        __syncwarp();
                    }
                    double2* cell = reinterpret_cast<double2*>(stg + (kOneBox ? 0 : (j2 >> 3) * 4096) + lane * 128 +
                                                               (((j2 & 7) ^ (lane & 7)) << 4));
                    double v0 = y[2 * j2], v1 = y[2 * j2 + 1];
                    const int ca = r0 + 2 * j2;
                    const double2 w2 = reinterpret_cast<const double2*>(wss)[j2];
                    v0 = dmul(w2.x, v0);
                    v1 = dmul(w2.y, v1);
                    if (POST == POST_XPROJ) {
                        if (ca < p.epi.split) v0 = softplus_d(dadd(v0, p.epi.bias[ca]));
                        if (ca + 1 < p.epi.split) v1 = softplus_d(dadd(v1, p.epi.bias[ca + 1]));
                    }
                    if (resid) {
                        const double2 x = *cell;
                        v0 = dadd(x.x, v0);
                        v1 = dadd(x.y, v1);
                    }
                    *cell = make_double2(v0, v1);
                }
                ptx::fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (kOneBox) {
                        ptx::tma_store_2d(om, stg, oc0 + 16, rbase);
                    } else {
                        ptx::tma_store_2d(om, stg, oc0, rbase);
                        ptx::tma_store_2d(om, stg + 4096, oc0 + 16, rbase);
                    }
                    ptx::bulk_commit();
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(acc_empty + buf);
                ptx::mbar_arrive(meta_empty + mslot);
            }
        }
        if (lane == 0) ptx::bulk_wait0();
    }
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc<2 * BN>(tmem_base);
}

// ---- int8 tensor-pipe probe (the INT8 peak is measured, not assumed) ----
// One CTA per SM; one thread issues `iters` x 4 back-to-back
// tcgen05.mma.cta_group::1.kind::i8 (M=128, N=256, K=32) on shared-memory
// operands into a TMEM accumulator, then commits once.
__global__ void __launch_bounds__(128, 1) k2_i8_probe(int iters) {
    __shared__ __align__(1024) uint8_t sb[256 * 128];  // operand values are irrelevant here:
    uint8_t* sa = sb;                                  // A aliases B's first 128 rows
    __shared__ uint64_t done;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<256>(&slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t d = slot;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = ptx::idesc_i8(128, 256);
        const uint64_t da = ptx::smem_desc_sw128(sa), db = ptx::smem_desc_sw128(sb);
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) ptx::mma_i8(d, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
        ptx::mma_commit(&done);
        ptx::mbar_wait(&done, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<256>(d);
}

double measure_i8_peak(cudaStream_t st, int num_sms) {
    const int iters = 8192;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k2_i8_probe<<<num_sms, 128, 0, st>>>(iters);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, st);
        k2_i8_probe<<<num_sms, 128, 0, st>>>(iters);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (cudaGetLastError() != cudaSuccess) return 0.0;
    const double ops = 2.0 * 128 * 256 * 32 * 4.0 * iters * num_sms;
    return ops / (best * 1e-3) / 1e12;
}

// ---- host side -------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

// 2-D int8 tensor [rows][cols] (cols contiguous), box = box_rows x 128 bytes, 128B swizzle.
static bool make_map(CUtensorMap* m, const void* base, int rows, int cols, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 2-D f64 tensor [rows][cols] (row pitch ld doubles): 32-row x 16-double boxes, 128B swizzle.
static bool make_map_f64(CUtensorMap* m, const double* base, int rows, int cols, int ld) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
    cuuint32_t box[2] = {16, 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 2-D packed A4 codes [rows][cols/2 bytes]: 128-row x 64-byte boxes, no swizzle (the
// unpack warps read them row-linear).
static bool make_map_packed(CUtensorMap* m, const void* base, int rows, int cols) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols / 2), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols / 2)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK / 2), static_cast<cuuint32_t>(kBM)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int BN, int EW, int POST, bool PLANES, bool PK, bool ONEBOX = false>
static cudaError_t launch_bn(const QLinParams& p, cudaStream_t st, int num_sms) {
    CUtensorMap ta, tb, to, to2;
    const bool amap = PK ? make_map_packed(&ta, p.a.codes4, p.M, p.K) : make_map(&ta, p.a.codes, p.M, p.K, kBM);
    if (!amap || !make_map(&tb, p.w, p.R, p.K, BN)) return cudaErrorInvalidValue;
    const bool inproj = p.epi.post == POST_INPROJ;
    const int ocols = inproj ? p.epi.split : p.R;
    if (!make_map_f64(&to, p.epi.out, p.M, ocols, p.epi.ld_out)) return cudaErrorInvalidValue;
    if (!make_map_f64(&to2, inproj ? p.epi.out2 : p.epi.out, p.M, inproj ? p.R - p.epi.split : ocols,
                      inproj ? p.epi.split : p.epi.ld_out))
        return cudaErrorInvalidValue;
    const int smem = K2Smem<BN, EW, ONEBOX>::kTotal;
    cudaError_t e = ensure_smem_attr<k2_qlinear<BN, EW, POST, PLANES, PK, ONEBOX>>(smem);
    if (e != cudaSuccess) return e;
    const int tiles = ((p.M + kBM - 1) / kBM) * ((p.R + BN - 1) / BN);
    const int grid = tiles < num_sms ? tiles : num_sms;
    k2_qlinear<BN, EW, POST, PLANES, PK, ONEBOX><<<grid, K2Cfg<EW, PK>::kThreads, smem, st>>>(ta, tb, to, to2, p);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

// Small M (at most two 128-row tiles, e.g. C1 at batch 1: 196 rows): the tensor-core
// pipeline's fill and drain (TMA, MMA, TMEM, TMA-store latency) is the whole launch, so
// one warp per (row, 32 output columns) computes the rows' int8 dot products with dp4a
// (exact int32 sums, any order) and runs the same f64 epilogue: S_m * acc, the outlier
// terms in ascending channel order (gemm.cpp:207-216), ws[r] * y, the post-op.
template <int POST, bool PLANES, bool PK>
__global__ void __launch_bounds__(128) k2_small(const QLinParams p) {
    constexpr int kRows = 1;  // rows per warp (4 rows sharing each weight load measured 8.2 vs 5.8 us: fewer warps)
    const int lane = threadIdx.x & 31;
    const long gw = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int nch = p.R / 32, mg = (p.M + kRows - 1) / kRows;
    if (gw >= static_cast<long>(mg) * nch) return;  // whole warps
    const int m0 = static_cast<int>(gw / nch) * kRows, r = static_cast<int>(gw % nch) * 32 + lane;
    const int K = p.K;
    const int8_t* __restrict__ wr = p.w + static_cast<size_t>(r) * K;
    const double wsr = p.ws[r];
    int acc[kRows];
    int mr[kRows];  // the rows (clamped: a ragged last group recomputes row M-1, stores skipped)
#pragma unroll
    for (int q = 0; q < kRows; ++q) {
        acc[q] = 0;
        mr[q] = min(m0 + q, p.M - 1);
    }
#pragma unroll 2
    for (int k = 0; k < K; k += 16) {
        const int4 wv = *reinterpret_cast<const int4*>(wr + k);
#pragma unroll
        for (int q = 0; q < kRows; ++q) {
            int4 cv;
            if constexpr (PK) {
                const uint2 c4 = *reinterpret_cast<const uint2*>(p.a.codes4 + static_cast<size_t>(mr[q]) * (K / 2) + k / 2);
                uint32_t c0, c1, c2, c3;
                unpack_nibbles8(c4.x, c0, c1);
                unpack_nibbles8(c4.y, c2, c3);
                cv = make_int4(static_cast<int>(c0), static_cast<int>(c1), static_cast<int>(c2), static_cast<int>(c3));
            } else {
                cv = *reinterpret_cast<const int4*>(p.a.codes + static_cast<size_t>(mr[q]) * K + k);
            }
            acc[q] = __dp4a(cv.x, wv.x, acc[q]);
            acc[q] = __dp4a(cv.y, wv.y, acc[q]);
            acc[q] = __dp4a(cv.z, wv.z, acc[q]);
            acc[q] = __dp4a(cv.w, wv.w, acc[q]);
        }
    }
#pragma unroll 1
    for (int q = 0; q < kRows; ++q) {
        const int m = m0 + q;
        if (m >= p.M) break;
        double y = dmul(p.a.s_row[m], i32_to_f64(static_cast<uint32_t>(acc[q])));
        int aout = 0;
        const int cnt = p.a.ocnt[m];
        if (cnt > 0) {  // outlier terms in ascending channel order (gemm.cpp:208-216)
            const uint32_t* mrow = p.a.omask + static_cast<size_t>(m) * p.a.J;
            int seen = 0;
            for (int wd = 0; wd < p.a.J && seen < cnt; ++wd) {
                unsigned bits = mrow[wd];
                while (bits) {
                    const int ch = wd * 32 + __ffs(bits) - 1;
                    bits &= bits - 1;
                    ++seen;
                    const size_t oi = static_cast<size_t>(m) * K + ch;
                    const int xo_i = p.a.ocode[oi];
                    const int wq = wr[ch];
                    const double coeff = dmul(p.a.oscale[oi], i32_to_f64(static_cast<uint32_t>(wq)));
                    y = dadd(y, dmul(coeff, i32_to_f64(static_cast<uint32_t>(xo_i))));
                    if (PLANES) aout += wq * xo_i;
                }
            }
        }
        if (PLANES) {
            p.epi.acc_in[static_cast<size_t>(m) * p.R + r] = acc[q];
            p.epi.acc_out[static_cast<size_t>(m) * p.R + r] = aout;
        }
        double v = dmul(wsr, y);
        if (POST == POST_XPROJ && r < p.epi.split) v = softplus_d(dadd(v, p.epi.bias[r]));
        double* dst = (POST == POST_INPROJ && r >= p.epi.split)
                          ? p.epi.out2 + static_cast<size_t>(m) * p.epi.split + (r - p.epi.split)
                          : p.epi.out + static_cast<size_t>(m) * p.epi.ld_out + r;
        if (POST == POST_RESID) v = dadd(*dst, v);
        *dst = v;
    }
}

template <int POST, bool PLANES, bool PK>
static cudaError_t launch_small_m(const QLinParams& p, cudaStream_t st) {
    const long warps = static_cast<long>(p.M) * (p.R / 32);
    k2_small<POST, PLANES, PK><<<static_cast<unsigned>((warps * 32 + 127) / 128), 128, 0, st>>>(p);
    ++kernel_launch_counter();
    return cudaGetLastError();
}

cudaError_t launch_qlinear(const QLinParams& p, cudaStream_t st, int num_sms) {
    if (p.M < 1 || p.R < 1 || p.K < 1 || (p.K % 16) != 0 || (p.R % 16) != 0) return cudaErrorInvalidValue;
    if (p.epi.post == POST_INPROJ && (p.epi.split % 32) != 0) return cudaErrorInvalidValue;
    if ((p.epi.ld_out % 2) != 0 || (p.R % 32) != 0) return cudaErrorInvalidValue;  // TMA pitch, whole chunks
    if (p.a.J < (p.K + 31) / 32) return cudaErrorInvalidValue;
    const bool pk = p.a.codes4 != nullptr;
    if (pk ? (p.K % 32) != 0 : p.a.codes == nullptr) return cudaErrorInvalidValue;  // packed rows: 16-byte pitch
    const bool planes = p.epi.acc_in != nullptr && p.epi.acc_out != nullptr;
    if (planes != (p.epi.acc_in != nullptr || p.epi.acc_out != nullptr)) return cudaErrorInvalidValue;
    // The packed-A4 operand adds an unpack warpgroup; it runs on the 8-epilogue-warp shape only
    // (16 epilogue warps + 4 unpack warps: 768 threads leave a per-CTA register pool of 80 x 768,
    // too small for the 104-register epilogue after setmaxnreg)
    // 16 epilogue warps with one staging box and 4 stages for calls of at least a wave of tiles
    // with K <= 1024 and no residual; below a wave (the box reuse's serialisation shows) and
    // for K > 1024 (the 8-warp shape's hoisted / vectorised outlier walk) the earlier rule:
    // 8 epilogue warps and 4 stages for wide R, else 16 epilogue warps and 2 stages
    // (profiles/r02/c5_quant_linear_r02q.txt)
    const long tiles = static_cast<long>((p.M + kBM - 1) / kBM) * ((p.R + 127) / 128);
    const bool onebox = p.epi.post != POST_RESID && p.K <= 1024 && tiles >= num_sms;
    const bool wide = p.epi.post != POST_RESID && (p.R > 512 || p.K > 1024);
    // at most two 128-row tiles: the dp4a kernel (M = 196 at batch 1: 5.8 vs 9.3 us per launch)
    const bool small = p.M <= 2 * kBM;
#define K2_CASE(P)                                                                                       \
    case P:                                                                                              \
        if (small)                                                                                       \
            return pk ? (planes ? launch_small_m<P, true, true>(p, st) : launch_small_m<P, false, true>(p, st))    \
                      : (planes ? launch_small_m<P, true, false>(p, st) : launch_small_m<P, false, false>(p, st)); \
        if (pk)                                                                                          \
            return planes ? launch_bn<128, 8, P, true, true>(p, st, num_sms)                             \
                          : launch_bn<128, 8, P, false, true>(p, st, num_sms);                           \
        if (onebox)                                                                                      \
            return planes ? launch_bn<128, 16, P, true, false, P != POST_RESID>(p, st, num_sms)          \
                          : launch_bn<128, 16, P, false, false, P != POST_RESID>(p, st, num_sms);        \
        if (wide)                                                                                        \
            return planes ? launch_bn<128, 8, P, true, false>(p, st, num_sms)                            \
                          : launch_bn<128, 8, P, false, false>(p, st, num_sms);                          \
        return planes ? launch_bn<128, 16, P, true, false>(p, st, num_sms)                               \
                      : launch_bn<128, 16, P, false, false>(p, st, num_sms);
    switch (p.epi.post) {
        K2_CASE(POST_STORE)
        K2_CASE(POST_INPROJ)
        K2_CASE(POST_RESID)
        K2_CASE(POST_XPROJ)
        default: return cudaErrorInvalidValue;
    }
#undef K2_CASE
}

}  // namespace ob
