// odf_kernels.cuh -- sm_100a kernels of the oblivious-forest hot path (templates;
// instantiated by odf_k_*.cu, one kernel family per translation unit so they build in parallel).
//
//   K1 binarize   fp32 factors (TMA-staged, 128B-swizzled tiles) -> uint8 bins
//   K2 apply      bins -> per-document fp32 scores
//   K3 fused      K1 o K2 per 128-document tile; bins live only in shared memory
//   K6 index      leaf-index export / per-document FNV-1a fingerprint (tests)
//
// Paper: arxiv 2205.07307.  Node condition FACTOR[INDEX] < THRESHOLD
// (P:80); leaf index = the level conditions written as a binary number, true = 1
// (P:114-116), level l = bit l; score = sum over trees.  The
// binarized form is the north_star's uint8 bin = #{borders <= x}.
//
// One CTA = 16 consumer warps + 1 producer warp, persistent over 128-document
// tiles.  The producer streams, through one ring of shared-memory slots guarded
// by mbarriers, first the tile's factor sub-tiles (cp.async.bulk.tensor, TMA)
// and then the forest's tree chunks (cp.async.bulk), so the next tile's HBM
// reads start while the current tile's trees are still being applied.
//
// Exactness: every comparison is IEEE fp32 (no fast-math, no FTZ); index
// assembly is integer-exact; the fp32 summation order is fixed (DESIGN.md
// "Summation order"): group g = t mod 16 sums its trees in ascending order, and
// score = (((P_0 + P_1) + P_2) + ... + P_15).  Every kernel here uses that order.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <type_traits>

#pragma once
#include "odf_internal.h"

#ifndef ODF_DIAG
#define ODF_DIAG 0  // diagnostics builds (tools/, never the product): see build.build_variant
#endif

namespace odf {

#if ODF_DIAG & 8  // diagnostics build only: per-warp phase timeline (tools/timeline.py)
constexpr int kDiagIt = 64;  // tile iterations recorded per CTA
static __device__ unsigned long long g_diag[148 * kDiagIt * 16 * 8];
__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define DIAG_T(var) const unsigned long long var = gtime()
#else
#define DIAG_T(var)
#endif

// ---------------------------------------------------------------------------
// Shared memory: one dynamic buffer, addressed by byte OFFSETS from its start.
// Plain C++ loads/stores (compiler-schedulable LDS/STS); the asynchronous
// proxy (TMA, bulk copies, mbarriers) gets the absolute shared-window address.
// The buffer is 1024-byte aligned in the shared window (checked at kernel
// start), which the 128B TMA swizzle and the 256-byte leaf-table trick need.
// ---------------------------------------------------------------------------
extern __shared__ __align__(1024) uint8_t smem_raw[];

__device__ __forceinline__ uint32_t smem_addr(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t sabs(uint32_t off) { return smem_addr(smem_raw) + off; }
template <class T>
__device__ __forceinline__ T sld(uint32_t off)
{
    return *reinterpret_cast<const T *>(smem_raw + off);
}
template <class T>
__device__ __forceinline__ void sst(uint32_t off, T v)
{
    *reinterpret_cast<T *>(smem_raw + off) = v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) { return sld<uint32_t>(a); }
__device__ __forceinline__ float lds_f32(uint32_t a) { return sld<float>(a); }
__device__ __forceinline__ uint2 lds_v2u(uint32_t a) { return sld<uint2>(a); }
__device__ __forceinline__ uint4 lds_v4u(uint32_t a) { return sld<uint4>(a); }
__device__ __forceinline__ float4 lds_v4f(uint32_t a) { return sld<float4>(a); }
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) { sst<uint8_t>(a, static_cast<uint8_t>(v)); }
__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) { sst<uint32_t>(a, v); }
__device__ __forceinline__ void sts_v4f(uint32_t a, float x, float y, float z, float w)
{
    sst<float4>(a, make_float4(x, y, z, w));
}
__device__ __forceinline__ void sts_v4u(uint32_t a, uint4 v) { sst<uint4>(a, v); }
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
// Loads by ABSOLUTE shared-window address (stage 1: read-only TMA-slot data, so
// volatile asm keeps them after the slot's mbarrier wait; ptxas still schedules
// them and folds constant offsets into the LDS immediate).
__device__ __forceinline__ uint32_t ldsa_u32(uint32_t a)
{
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ uint32_t ldsa_u16(uint32_t a)
{
    uint16_t r;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ float ldsa_f32(uint32_t a)
{
    float r;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(a));
    return r;
}
__device__ __forceinline__ float4 ldsa_v4f(uint32_t a)
{
    float4 r;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "r"(a));
    return r;
}
__device__ __forceinline__ uint4 ldsa_v4u(uint32_t a)
{
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(a));
    return r;
}
__device__ __forceinline__ void named_bar_consumers()
{
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerThreads) : "memory");
}
// mbarriers / bulk copies: arguments are buffer OFFSETS
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sabs(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sabs(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sabs(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(sabs(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "ODF_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra ODF_WAIT_%=;\n}\n" ::"r"(sabs(bar)),
        "r"(parity), "n"(0x989680)  // suspend-time hint: the warp sleeps instead of spinning
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(sabs(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(sabs(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(sabs(dst)),
        "l"(src), "r"(bytes), "r"(sabs(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, uint32_t src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(sabs(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all()
{
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all()
{
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Stage 1: binarization of one 128-doc x 32-factor sub-tile
// ---------------------------------------------------------------------------
// The TMA box lands with SWIZZLE_128B: 16-byte chunk q of row r sits at chunk
// q ^ (r & 7), so warp-wide reads of one chunk (32 rows) are conflict-free.
// A warp handles one factor quad q (the 4 factors of chunk q, read with one
// LDS.128 per document) for NDL documents per lane: dbase + lane + 32n.
//
// bin(x) = #{j : !(x < b_j)}.  The quad is two pairs of adjacent
// factors; both factors of a pair share one code path chosen by the model
// compiler (fmeta.y & 0xf, warp-uniform):
//   LIN4  both m <= 4: count !(x < e_j) over 4 entries (one broadcast LDS.128
//         per factor, no dependent chain);
//   BIN L branchless search over a sorted array of 2^L - 1 entries, stored skewed
//         (position p at p + (p >> 5)) so the lanes of one step hit distinct banks;
//         the pair's 2*NDL chains run interleaved.
// Every array is the factor's sorted borders PRECEDED by npad = (length - m)
// copies of -inf.  !(x < -inf) holds for every x (NaN included), so the count over
// the padded array is exactly npad + bin(x): bin = count - npad, no clamping.
// An unused factor of a pair searches its partner's array and stores into the
// trash column.  In the fused/latency paths a factor with m > 127 borders stores
// C = ceil(m / 127) 7-bit code columns (fmeta.y bits 4-7 = C - 1): column c holds
// clamp(bin - 127c, 0, 127), so a level on border k tests column k / 127 against
// k % 127.  The binarize kernel stores true bins: u8,
// or u16 for "wide" models (some factor with > 254 borders, NEXT-4).
enum : uint32_t { CLS_SKIP = 0, CLS_LIN4 = 1 };  // cls >= 2: BIN with L = cls - 1
constexpr uint32_t kExtraShift = 4;              // fmeta.y bits 4-7: code columns - 1
constexpr uint32_t kPairSplit = 1u << 8;         // fmeta.y of a pair's first factor: a factor of
                                                 // the pair has > 127 borders (two code columns)

__host__ __device__ constexpr uint32_t skew(uint32_t p) { return p + (p >> 5); }

// 0xffffffff if !(x < b) (unordered or >=: NaN counts), else 0
__device__ __forceinline__ uint32_t not_less_mask(float x, float b)
{
    uint32_t r;
    asm("set.geu.u32.f32 %0, %1, %2;" : "=r"(r) : "f"(x), "f"(b));
    return r;
}
// v += inc if !(x < b) (unordered or >=): one FSETP + one predicated IADD
__device__ __forceinline__ void add_if_not_less(uint32_t &v, float x, float b, uint32_t inc)
{
    asm("{\n\t.reg .pred p;\n\tsetp.geu.f32 p, %1, %2;\n\t@p add.u32 %0, %0, %3;\n\t}"
        : "+r"(v)
        : "f"(x), "f"(b), "r"(inc));
}

// fmeta.y bits 16-31 hold -npad (two's complement, 16 bits)
__device__ __forceinline__ uint32_t neg_npad(const uint4 &m)
{
    return static_cast<uint32_t>(static_cast<int32_t>(m.y) >> 16);
}

// Where the bins / codes of a tile go: shared memory (fused, binarize) or a
// global [n_cols + 1][128] block (latency path).
// Every sink also has stn(off, v[NDL]): v[n] at off + 32n (the NDL documents of a lane).
struct SmemSink {
    uint32_t base;
    __device__ __forceinline__ void st(uint32_t off, uint32_t v) const { sts_u8(base + off, v); }
    template <int NDL>
    __device__ __forceinline__ void stn(uint32_t off, const uint32_t (&v)[NDL]) const
    {
#pragma unroll
        for (int n = 0; n < NDL; ++n) sts_u8(base + off + 32u * n, v[n]);
    }
    __device__ __forceinline__ SmemSink at(uint32_t off) const { return SmemSink{base + off}; }
};
struct GmemSink {
    uint8_t *base;
    __device__ __forceinline__ void st(uint32_t off, uint32_t v) const
    {
        base[off] = static_cast<uint8_t>(v);
    }
    template <int NDL>
    __device__ __forceinline__ void stn(uint32_t off, const uint32_t (&v)[NDL]) const
    {
        uint8_t *q = base + off;
#pragma unroll
        for (int n = 0; n < NDL; ++n) q[32 * n] = static_cast<uint8_t>(v[n]);
    }
};
// The binarize kernel (K1) writes each warp's bins straight to the tile's block of
// the blocked bins layout in HBM (row u = used factor u at offset u * tile docs):
// 32 lanes store 32 consecutive bytes per instruction; offsets >= limit (the trash
// column of unused pair slots) are dropped.
struct GmemBinsSink {
    uint8_t *base;
    uint32_t limit;
    __device__ __forceinline__ void st(uint32_t off, uint32_t v) const
    {
        if (off < limit) base[off] = static_cast<uint8_t>(v);
    }
    // one bound test and one 64-bit address per factor; the documents 32 apart are
    // immediate offsets of the same address
    template <int NDL>
    __device__ __forceinline__ void stn(uint32_t off, const uint32_t (&v)[NDL]) const
    {
        if (off < limit) {
            uint8_t *q = base + off;
#pragma unroll
            for (int n = 0; n < NDL; ++n) q[32 * n] = static_cast<uint8_t>(v[n]);
        }
    }
};
struct GmemBinsSink16 {  // wide models: u16 bins
    uint16_t *base;
    uint32_t limit;
    __device__ __forceinline__ void st(uint32_t off, uint32_t v) const
    {
        if (off < limit) base[off] = static_cast<uint16_t>(v);
    }
    template <int NDL>
    __device__ __forceinline__ void stn(uint32_t off, const uint32_t (&v)[NDL]) const
    {
        if (off < limit) {
            uint16_t *q = base + off;
#pragma unroll
            for (int n = 0; n < NDL; ++n) q[32 * n] = static_cast<uint16_t>(v[n]);
        }
    }
};

// u16 true bins of a wide model (binarize kernel): element offsets, 2 bytes each
struct SmemSink16 {
    uint32_t base;
    __device__ __forceinline__ void st(uint32_t off, uint32_t v) const
    {
        sst<uint16_t>(base + 2u * off, static_cast<uint16_t>(v));
    }
    template <int NDL>
    __device__ __forceinline__ void stn(uint32_t off, const uint32_t (&v)[NDL]) const
    {
#pragma unroll
        for (int n = 0; n < NDL; ++n) st(off + 32u * n, v[n]);
    }
    __device__ __forceinline__ SmemSink16 at(uint32_t off) const { return SmemSink16{base + off}; }
};

// Both factors of a pair: one warp-uniform test for code-column splits per pair.
template <int NDL, bool CODES, class Sink>
__device__ __forceinline__ void store_pair(const Sink &s, const uint4 &ma, const uint4 &mb, uint32_t d0,
                                           const uint32_t (&ra)[NDL], const uint32_t (&rb)[NDL]);

template <int NDL, bool CODES, class Sink>
__device__ __forceinline__ void store_bins(const Sink &s, const uint4 &m, uint32_t d0,
                                           const uint32_t (&bin)[NDL])
{
    // extra code columns: 0 or 1 here (factors with > 254 borders are searched by
    // bin_pair_wide, which stores any number of columns)
    if (CODES && (m.y & (1u << kExtraShift))) {  // 128..254 borders: code columns A and B
#pragma unroll
        for (int n = 0; n < NDL; ++n) {
            s.st(m.z + d0 + 32 * n, min(bin[n], 127u));
            s.st(m.w + d0 + 32 * n, max(bin[n], 127u) - 127u);
        }
    } else {
        s.template stn<NDL>(m.z + d0, bin);
    }
}

template <int NDL, bool CODES, class Sink>
__device__ __forceinline__ void store_pair(const Sink &s, const uint4 &ma, const uint4 &mb, uint32_t d0,
                                           const uint32_t (&ra)[NDL], const uint32_t (&rb)[NDL])
{
    if (CODES && (ma.y & kPairSplit)) {
        store_bins<NDL, CODES>(s, ma, d0, ra);
        store_bins<NDL, CODES>(s, mb, d0, rb);
    } else {
        s.template stn<NDL>(ma.z + d0, ra);
        s.template stn<NDL>(mb.z + d0, rb);
    }
}

// Any number of 7-bit code columns A, B0, B1, ... (B contiguous): column c holds
// clamp(bin - 127c, 0, 127) (wide pairs only).
template <int NDL, bool CODES, class Sink>
__device__ __forceinline__ void store_bins_any(const Sink &s, const uint4 &m, uint32_t d0,
                                               const uint32_t (&bin)[NDL])
{
    const uint32_t extra = CODES ? (m.y >> kExtraShift) & 0xfu : 0u;  // warp-uniform
#pragma unroll
    for (int n = 0; n < NDL; ++n) {
        s.st(m.z + d0 + 32 * n, extra ? min(bin[n], 127u) : bin[n]);
#pragma unroll 1
        for (uint32_t c = 1; c <= extra; ++c)
            s.st(m.w + (c - 1u) * kTile + d0 + 32 * n, min(max(bin[n], 127u * c) - 127u * c, 127u));
    }
}

template <int NDL, bool CODES, class Sink>
__device__ __forceinline__ void lin4_pair(const float (&xa)[NDL], const float (&xb)[NDL],
                                          const uint4 &ma, const uint4 &mb, uint32_t bord,
                                          const Sink &s, uint32_t d0)
{
    const float4 ea = ldsa_v4f(bord + ma.x), eb = ldsa_v4f(bord + mb.x);
    const uint32_t na = neg_npad(ma), nb = neg_npad(mb);
    uint32_t ra[NDL], rb[NDL];
#pragma unroll
    for (int n = 0; n < NDL; ++n) {
        ra[n] = na;
        rb[n] = nb;
        add_if_not_less(ra[n], xa[n], ea.x, 1u);
        add_if_not_less(rb[n], xb[n], eb.x, 1u);
        add_if_not_less(ra[n], xa[n], ea.y, 1u);
        add_if_not_less(rb[n], xb[n], eb.y, 1u);
        add_if_not_less(ra[n], xa[n], ea.z, 1u);
        add_if_not_less(rb[n], xb[n], eb.z, 1u);
        add_if_not_less(ra[n], xa[n], ea.w, 1u);
        add_if_not_less(rb[n], xb[n], eb.w, 1u);
    }
    store_pair<NDL, CODES>(s, ma, mb, d0, ra, rb);
}

template <int L>
__device__ __forceinline__ uint32_t pos_to_bin(uint32_t pos, uint32_t base, uint32_t nnpad)
{
    if constexpr (L <= 5) {
        return (pos - base + 4u * nnpad) >> 2;  // count >= npad always
    } else {
        uint32_t idx = (pos - base) >> 2;
        idx -= idx / 33u;  // unskew: s = p + p/32 -> p = s - s/33 (exact)
        return idx + nnpad;
    }
}

template <int L, int NDL, bool CODES, class Sink>
__device__ __forceinline__ void bin_pair(const float (&xa)[NDL], const float (&xb)[NDL],
                                         const uint4 &ma, const uint4 &mb, uint32_t bord,
                                         const Sink &s, uint32_t d0)
{
    const uint32_t a0 = bord + ma.x, b0 = bord + mb.x;
    uint32_t pa[NDL], pb[NDL];
#pragma unroll
    for (int n = 0; n < NDL; ++n) {
        pa[n] = a0;
        pb[n] = b0;
    }
#pragma unroll
    for (int st = L - 1; st >= 0; --st) {
        const uint32_t w = 1u << st;
        float ea[NDL], eb[NDL];
#pragma unroll
        for (int n = 0; n < NDL; ++n) {
            ea[n] = ldsa_f32(pa[n] + 4u * skew(w - 1));
            eb[n] = ldsa_f32(pb[n] + 4u * skew(w - 1));
        }
#pragma unroll
        for (int n = 0; n < NDL; ++n) {
            add_if_not_less(pa[n], xa[n], ea[n], 4u * (w + (w >> 5)));
            add_if_not_less(pb[n], xb[n], eb[n], 4u * (w + (w >> 5)));
        }
    }
    uint32_t ra[NDL], rb[NDL];
#pragma unroll
    for (int n = 0; n < NDL; ++n) {
        ra[n] = pos_to_bin<L>(pa[n], a0, neg_npad(ma));
        rb[n] = pos_to_bin<L>(pb[n], b0, neg_npad(mb));
    }
    store_pair<NDL, CODES>(s, ma, mb, d0, ra, rb);
}

// Wide factors (L = 9..11: > 254 borders or paired with such; NEXT-4): the same search with a run-time
// step count (one compact loop instead of three unrolled copies in the I-cache).
template <int NDL, bool CODES, class Sink>
__device__ __forceinline__ void bin_pair_wide(const float (&xa)[NDL], const float (&xb)[NDL],
                                           const uint4 &ma, const uint4 &mb, uint32_t bord,
                                           const Sink &s, uint32_t d0, uint32_t L)
{
    const uint32_t a0 = bord + ma.x, b0 = bord + mb.x;
    uint32_t pa[NDL], pb[NDL];
#pragma unroll
    for (int n = 0; n < NDL; ++n) {
        pa[n] = a0;
        pb[n] = b0;
    }
#pragma unroll 1
    for (int st = static_cast<int>(L) - 1; st >= 0; --st) {
        const uint32_t w = 1u << st, off = 4u * skew(w - 1), inc = 4u * (w + (w >> 5));
        float ea[NDL], eb[NDL];
#pragma unroll
        for (int n = 0; n < NDL; ++n) {
            ea[n] = ldsa_f32(pa[n] + off);
            eb[n] = ldsa_f32(pb[n] + off);
        }
#pragma unroll
        for (int n = 0; n < NDL; ++n) {
            add_if_not_less(pa[n], xa[n], ea[n], inc);
            add_if_not_less(pb[n], xb[n], eb[n], inc);
        }
    }
    uint32_t ra[NDL], rb[NDL];
#pragma unroll
    for (int n = 0; n < NDL; ++n) {
        ra[n] = pos_to_bin<11>(pa[n], a0, neg_npad(ma));
        rb[n] = pos_to_bin<11>(pb[n], b0, neg_npad(mb));
    }
    store_bins_any<NDL, CODES>(s, ma, d0, ra);
    store_bins_any<NDL, CODES>(s, mb, d0, rb);
}

template <int NDL, bool CODES, bool WIDE, class Sink>
__device__ __forceinline__ void bin_pair_dispatch(const float (&xa)[NDL], const float (&xb)[NDL],
                                                  const uint4 &ma, const uint4 &mb, uint32_t bord,
                                                  const Sink &s, uint32_t d0)
{
    // warp-uniform class; an if-chain ordered by frequency instead of a jump table
    // (cls 2, 3 = BIN 1, 2 never occur: pairs with <= 4 borders are LIN4)
    const uint32_t cls = ma.y & 0xfu;
    if (cls == CLS_LIN4) {
        lin4_pair<NDL, CODES>(xa, xb, ma, mb, bord, s, d0);
    } else if (cls == CLS_SKIP) {
    } else if (cls <= 5) {
        if (cls == 5) bin_pair<4, NDL, CODES>(xa, xb, ma, mb, bord, s, d0);
        else bin_pair<3, NDL, CODES>(xa, xb, ma, mb, bord, s, d0);
    } else if (cls <= 7) {
        if (cls == 6) bin_pair<5, NDL, CODES>(xa, xb, ma, mb, bord, s, d0);
        else bin_pair<6, NDL, CODES>(xa, xb, ma, mb, bord, s, d0);
    } else if (cls <= 9) {
        if (cls == 8) bin_pair<7, NDL, CODES>(xa, xb, ma, mb, bord, s, d0);
        else bin_pair<8, NDL, CODES>(xa, xb, ma, mb, bord, s, d0);
    } else if constexpr (WIDE) {  // models with > 254 borders on some factor only
        bin_pair_wide<NDL, CODES>(xa, xb, ma, mb, bord, s, d0, cls - 1u);
    }
}

// tile: the 16 KB factor box; meta: its 32 fmeta entries (512 B); bord: its
// factors' border arrays (fmeta.x is relative to bord) -- all in the TMA slot,
// given as buffer offsets.  Quad q, documents d0 + 32n (n < NDL), d0 = dbase + lane.
// CSH: code-column shift.  The model compiler bakes column offsets as col * 128; a
// 64-document tile (2 documents per lane, DPL = 2) lays its columns 64 bytes apart.
template <int NDL, bool CODES, bool WIDE, bool FM, class Sink, int CSH = 0>
__device__ __forceinline__ void binarize_sub(uint32_t tile, uint32_t meta, uint32_t bord,
                                             const Sink &bins, int q, int dbase, int lane)
{
    const uint32_t ma_ = sabs(meta) + 64u * q;
    uint4 m0 = ldsa_v4u(ma_), m2 = ldsa_v4u(ma_ + 32u);
    if (((m0.y | m2.y) & 0xfu) == CLS_SKIP) return;  // warp-uniform: no used factor in the quad
    uint4 m1 = ldsa_v4u(ma_ + 16u), m3 = ldsa_v4u(ma_ + 48u);
    if constexpr (CSH != 0) {
        m0.z >>= CSH; m0.w >>= CSH; m1.z >>= CSH; m1.w >>= CSH;
        m2.z >>= CSH; m2.w >>= CSH; m3.z >>= CSH; m3.w >>= CSH;
    }
    const uint32_t d0 = static_cast<uint32_t>(dbase + lane);
    const uint32_t ta = sabs(tile), ba = sabs(bord);
    float x[4][NDL];
#pragma unroll
    for (int n = 0; n < NDL; ++n) {
        const uint32_t d = d0 + 32u * n;
        float4 v;
        if constexpr (FM) {  // feature-major box [32 factors][tile docs]: lanes = docs
            constexpr uint32_t RB = 512u >> CSH;  // row bytes
            const uint32_t r = ta + q * 4 * RB + d * 4;
            v = make_float4(ldsa_f32(r), ldsa_f32(r + RB), ldsa_f32(r + 2 * RB), ldsa_f32(r + 3 * RB));
        } else {   // doc-major box [128 docs][32 factors], 128B-swizzled (d & 7 == lane & 7)
            v = ldsa_v4f(ta + d * 128 + ((q ^ (lane & 7)) << 4));
        }
        x[0][n] = v.x;
        x[1][n] = v.y;
        x[2][n] = v.z;
        x[3][n] = v.w;
    }
    bin_pair_dispatch<NDL, CODES, WIDE>(x[0], x[1], m0, m1, ba, bins, d0);
    bin_pair_dispatch<NDL, CODES, WIDE>(x[2], x[3], m2, m3, ba, bins, d0);
}

// ---------------------------------------------------------------------------
// Stage 2: leaf-index assembly (SWAR, 4 documents per lane)
// ---------------------------------------------------------------------------
// Lane j holds documents 4j..4j+3 of the tile as the 4 bytes of one u32 read
// from the bins row of a column.  Codes are 7-bit (factors with > 127 borders
// use two columns), so for a level with descriptor (col, 128-K) the
// byte sum code + (128 - K) (the byte replicated by one PRMT) never carries out
// of its byte and its bit 7 is the "flag" code >= K, i.e. the condition is
// FALSE.  Flags are shifted in from the top of each byte, so after DEPTH levels
// level l sits at bit 8-DEPTH+l: the byte is the complemented leaf index F,
// and leaf tables are stored reversed (table[F] = leaf[2^d-1-F]).
// Descriptors (odf_internal.h): depth <= 8 the split format (column words, then the
// K bytes packed four per word: a depth-6 tree is 32 B = two warp-uniform LDS.128);
// depth 9-10 one 4-byte word per level.
// A lane's view of a tile's code block: the absolute address of its 4 documents'
// bytes in code column 0.
struct Lane {
    uint32_t bins;
};
__device__ __forceinline__ Lane make_lane(const KParams &, uint32_t bins_abs) { return Lane{bins_abs}; }
// One level: the lane's code word of the level's column, and the byte-wise
// "code >= K" flags in bit 7 (code + (128 - K) never carries out of its byte),
// shifted into the index.  (Moving the address / merge onto the FMA pipe with
// IMAD.HI was tried: SASS IMAD.HI takes a 64-bit addend, so every merge needs a
// register-pair set-up and the FMA pipe became the binder.)
// The lane's code word: 4 documents (u32) or, 64-document tiles, 2 (u16, upper bytes
// 0: their sums stay below 128, so their flags are 0 and never used).
template <int DPL>
__device__ __forceinline__ uint32_t code_word(uint32_t a)
{
    if constexpr (DPL == 4) return ldsa_u32(a);
    else return ldsa_u16(a);
}

// One level's flags: the lane's code word of the level's column, and the byte-wise
// "code >= K" flags in bit 7 of each byte (code + (128 - K) never carries out of its
// byte); krep = (128 - K) in every byte.
template <int DPL = 4>
__device__ __forceinline__ uint32_t level_flags(uint32_t col128, uint32_t krep, const Lane &ln)
{
    return (code_word<DPL>(ln.bins + (DPL == 4 ? col128 : col128 >> 1)) + krep) & 0x80808080u;
}
// OR_j f[j] >> (N-1-j) from independent pairs (f[j] >> 1 | f[j+1]), then merged
// pair by pair: a shorter dependency chain than N serial shift-or steps (c3 fused
// -0.9 %, c2 -2.7 %; the pairing measured better than a halving tree on c3 apply)
template <int N>
__device__ __forceinline__ uint32_t merge_flags(const uint32_t *f)
{
    if constexpr (N <= 0) {
        return 0u;
    } else if constexpr (N == 1) {
        return f[0];
    } else {
        constexpr int H = N > 2 ? 2 : 1;
        return (merge_flags<N - H>(f) >> H) | merge_flags<H>(f + (N - H));
    }
}

// Split-format descriptors of one tree, in registers (odf_internal.h): column
// words, then K bytes; loaded as LDS.128 groups, the tail as LDS.64 / LDS.32.
template <int DEPTH>
struct SplitDesc {
    static constexpr int NW = desc_split_words(DEPTH);
    uint32_t w[NW > 0 ? (NW + 3) & ~3 : 1];
};
template <int DEPTH>
__device__ __forceinline__ SplitDesc<DEPTH> load_split(uint32_t d)
{
    SplitDesc<DEPTH> s;
    constexpr int NW = SplitDesc<DEPTH>::NW;
#pragma unroll
    for (int g = 0; g < NW; g += 4) {
        if (g + 2 < NW) {
            const uint4 q = lds_v4u(d + g * 4);
            s.w[g] = q.x; s.w[g + 1] = q.y; s.w[g + 2] = q.z; s.w[g + 3] = q.w;
        } else if (g + 1 < NW) {
            const uint2 q = lds_v2u(d + g * 4);
            s.w[g] = q.x; s.w[g + 1] = q.y;
        } else {
            s.w[g] = lds_u32(d + g * 4);
        }
    }
    return s;
}

// The flags of every level of the tree whose descriptors start at d, merged into
// lo (levels 0..7: after all levels, level l of a depth-D tree sits at bit
// 8 - min(D,8) + l of each byte) and hi (levels 8..: level 8 + j at bit
// 16 - D + j); the byte of lo (| hi's bits above) is the complemented index F.
template <int DEPTH, int DPL = 4>
__device__ __forceinline__ void tree_flags(uint32_t d, const Lane &ln, uint32_t &lo,
                                           uint32_t &hi)
{
    uint32_t f[DEPTH > 0 ? DEPTH : 1];
    if constexpr (desc_fmt(DEPTH) == DESC_SPLIT) {
        const SplitDesc<DEPTH> sd = load_split<DEPTH>(d);
#pragma unroll
        for (int l = 0; l < DEPTH; ++l)
            f[l] = level_flags<DPL>(sd.w[l], prmt(sd.w[DEPTH + l / 4], 0u, 0x1111u * (l & 3)), ln);
    } else if constexpr (desc_fmt(DEPTH) == DESC8) {
#pragma unroll
        for (int l = 0; l < DEPTH; l += 2) {  // one LDS.128 per two levels
            const uint4 q = lds_v4u(d + l * 8);
            f[l] = level_flags<DPL>(q.x, q.y, ln);
            if (l + 1 < DEPTH) f[l + 1] = level_flags<DPL>(q.z, q.w, ln);
        }
    } else {
        // 4-byte descriptors: col * 128 = dsc >> 12, the byte 128 - K replicated by PRMT
        uint32_t w[DEPTH > 0 ? (DEPTH + 3) & ~3 : 1];
#pragma unroll
        for (int l = 0; l < DEPTH; l += 4) {
            if (l + 2 < DEPTH) {  // 3 or 4 levels left: one LDS.128 (padding levels unused)
                const uint4 q = lds_v4u(d + l * 4);
                w[l] = q.x; w[l + 1] = q.y; w[l + 2] = q.z; w[l + 3] = q.w;
            } else if (l + 1 < DEPTH) {
                const uint2 q = lds_v2u(d + l * 4);
                w[l] = q.x; w[l + 1] = q.y;
            } else {
                w[l] = lds_u32(d + l * 4);
            }
        }
#pragma unroll
        for (int l = 0; l < DEPTH; ++l) f[l] = level_flags<DPL>(w[l] >> 12, prmt(w[l], 0u, 0x0000u), ln);
    }
    constexpr int NLO = DEPTH < 8 ? DEPTH : 8;
    lo = merge_flags<NLO>(f);
    hi = merge_flags<DEPTH - NLO>(f + NLO);
}

// Complemented leaf index F of the lane's 4 documents.
template <int DEPTH, int DPL = 4>
__device__ __forceinline__ void tree_findex(uint32_t d, const Lane &ln, uint32_t F[DPL])
{
    uint32_t lo, hi;
    tree_flags<DEPTH, DPL>(d, ln, lo, hi);
#pragma unroll
    for (int n = 0; n < DPL; ++n) {
        if constexpr (DEPTH == 0) {
            F[n] = 0;
        } else if constexpr (DEPTH <= 8) {
            F[n] = ((lo >> (8 * n)) & 0xffu) >> (8 - DEPTH);
        } else {
            const uint32_t h = hi >> (16 - DEPTH);
            F[n] = ((lo >> (8 * n)) & 0xffu) | (((h >> (8 * n)) & 0xffu) << 8);
        }
    }
}

// Bank-swizzled leaf tables (model compiler: leaf_pos in odf_capi.cu).  A warp's
// 32 gathers from one table conflict when two lanes want different words of one
// bank; with 2^d > 32 words a bank holds several.  Leaf indices are skewed (a
// level's condition is mostly true or mostly false), so popular indices differ in
// few bits: the words sharing a bank are chosen FAR apart in Hamming distance.
// With F = H * 32 + L (L = the 5 low bits), word F is stored at bank
//   depth 6:      L ^ (H ? 31 : 0)          (F shares its bank only with F ^ 63)
//   depth 7..10:  L ^ H ^ (parity(H) ? 31 : 0)  (a [d, 5] code of distance 4: two
//                 indices in one bank differ in >= 4 bits)
// and row H.  Simulated on the c3/c4 models: 1.90 -> 1.21 (depth 6) and 5.5 ->
// 2.3 (depth 10) wavefronts per warp gather.  Here: 4 documents per lane, lo =
// F's low 8 bits per byte, h = F's bits 8.. per byte; rewrites lo's 5 low bits.
__device__ __forceinline__ uint32_t swz_bank_hi(uint32_t lo, uint32_t h)
{
    const uint32_t g = ((lo >> 5) & 0x07070707u) | (h << 3);  // H per byte (<= 5 bits)
    const uint32_t x = g ^ (g >> 1) ^ (g >> 2);                // bit 0: g0^g1^g2
    const uint32_t par = (x ^ (x >> 3)) & 0x01010101u;         // bit 0: parity(H)
    return lo ^ g ^ (par * 31u);
}

// Absolute shared-window addresses of the 4 leaves (tables reversed and
// bank-swizzled; tb = the table base, absolute and 256-aligned).
template <int DEPTH, int DPL = 4>
__device__ __forceinline__ void addrs_from_flags(uint32_t lo, uint32_t hi, uint32_t tb, uint32_t a[DPL])
{
    if constexpr (DEPTH <= 6) {
        // byte = F << (8-DEPTH); want 4F in the low byte of a 256-aligned base
        if constexpr (DEPTH < 6 && DEPTH > 0) lo >>= (6 - DEPTH);
        // depth 6: byte bit 7 = F bit 5 -> complement F's 5 low bits (byte bits 2..6)
        if constexpr (DEPTH == 6) lo ^= prmt(lo, 0u, 0xBA98u) & 0x7C7C7C7Cu;
#pragma unroll
        for (int n = 0; n < DPL; ++n) a[n] = prmt(lo, tb, 0x7650u | n);
    } else if constexpr (DEPTH <= 8) {
        if constexpr (DEPTH == 7) lo = (lo >> 1) & 0x7F7F7F7Fu;  // byte = F
        lo = swz_bank_hi(lo, 0u);
#pragma unroll
        for (int n = 0; n < DPL; ++n) a[n] = tb + (prmt(lo, 0u, 0x4440u | n) << 2);
    } else {
        const uint32_t h = hi >> (16 - DEPTH);
        lo = swz_bank_hi(lo, h);
#pragma unroll
        for (int n = 0; n < DPL; ++n)
            a[n] = tb + (prmt(lo, h, 0xCC00u | ((4u + n) << 4) | n) << 2);
    }
}
template <int DEPTH, int DPL = 4>
__device__ __forceinline__ void leaf_addrs(uint32_t d, const Lane &ln, uint32_t tb,
                                           uint32_t a[DPL])
{
    uint32_t lo, hi;
    tree_flags<DEPTH, DPL>(d, ln, lo, hi);
    addrs_from_flags<DEPTH, DPL>(lo, hi, tb, a);
}


// Per-lane accumulators of the 4 documents: fp32 leaves summed in fp32 (the
// north_star's path) or, for MatrixNet integer models, u32 leaves summed in u64
// (exact, order-free).
template <bool U32, int DPL = 4>
struct Acc;
template <int DPL>
struct Acc<false, DPL> {
    float v[DPL] = {};
    // x += a, y += b as one packed FADD2 (each lane an IEEE round-to-nearest add: the
    // same results as two FADDs)
    static __device__ __forceinline__ void add2(float &x, float &y, float a, float b)
    {
        asm("{\n\t.reg .b64 p, q;\n\tmov.b64 p, {%0, %1};\n\tmov.b64 q, {%2, %3};\n\t"
            "add.rn.f32x2 p, p, q;\n\tmov.b64 {%0, %1}, p;\n\t}"
            : "+f"(x), "+f"(y)
            : "f"(a), "f"(b));
    }
    // leaves at ABSOLUTE shared-window addresses a[n]
    __device__ __forceinline__ void add4(const uint32_t (&a)[DPL])
    {
        float g[DPL];
#pragma unroll
        for (int n = 0; n < DPL; ++n) g[n] = ldsa_f32(a[n]);
#pragma unroll
        for (int n = 0; n < DPL; n += 2) add2(v[n], v[n + 1], g[n], g[n + 1]);
    }
    // Force the accumulators (hence every gather of the chunk) to be complete before
    // what follows, i.e. before the mbarrier arrive that hands the slot back to the
    // producer (ptxas may otherwise sink the FADDs, leaving gathers in flight).
    __device__ __forceinline__ void pin(uint32_t scratch) const
    {
        // a store predicated on all accumulators (never taken in practice): the
        // store cannot issue before the FADDs, hence before the gathers returned,
        // and it is ordered before the (memory) arrive
        uint32_t x = 0;
#pragma unroll
        for (int n = 0; n < DPL; ++n) x ^= __float_as_uint(v[n]);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %0, 0x7fc00001;\n\t@p st.shared.u32 [%1], %0;\n\t}"
                     ::"r"(x), "r"(sabs(scratch)) : "memory");
    }
    static constexpr uint32_t kRed = kRedBytes;
    // reduction buffer [16 groups][tile_docs]: group g's partials of the lane's DPL
    // documents (doc0 = the first document's position in the tile)
    __device__ __forceinline__ void to_red(uint32_t red, int g, int doc0, int tile_docs) const
    {
        if constexpr (DPL == 4)
            sts_v4f(red + (g * tile_docs + doc0) * 4, v[0], v[1], v[2], v[3]);
        else
            sst<float2>(red + (g * tile_docs + doc0) * 4, make_float2(v[0], v[1]));
    }
};
template <int DPL>
struct Acc<true, DPL> {
    unsigned long long v[DPL] = {};
    __device__ __forceinline__ void add4(const uint32_t (&a)[DPL])
    {
#pragma unroll
        for (int n = 0; n < DPL; ++n) v[n] += ldsa_u32(a[n]);
    }
    __device__ __forceinline__ void pin(uint32_t scratch) const
    {
        unsigned long long x = 0;
#pragma unroll
        for (int n = 0; n < DPL; ++n) x ^= v[n];
        const uint32_t y = static_cast<uint32_t>(x);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %0, 0x7fc00001;\n\t@p st.shared.u32 [%1], %0;\n\t}"
                     ::"r"(y), "r"(sabs(scratch)) : "memory");
    }
    static constexpr uint32_t kRed = 2 * kRedBytes;
    __device__ __forceinline__ void to_red(uint32_t red, int g, int doc0, int tile_docs) const
    {
        const uint32_t a = red + (g * tile_docs + doc0) * 8;
        sst<ulonglong2>(a, make_ulonglong2(v[0], v[1]));
        if constexpr (DPL == 4) sst<ulonglong2>(a + 16, make_ulonglong2(v[2], v[3]));
    }
};

#ifndef ODF_SPLIT_MIN_DEPTH
#define ODF_SPLIT_MIN_DEPTH 7  // A/B builds: smallest depth whose fused phase A uses the warp-half split
#endif
#ifndef ODF_APPLY_UNROLL
#define ODF_APPLY_UNROLL 2
#endif
constexpr int kApplyUnroll = ODF_APPLY_UNROLL;  // trees in flight per warp

template <int DEPTH, bool U32, int DPL = 4>
__device__ __forceinline__ void apply_tree(uint32_t chunk, uint32_t desc_bytes, const Lane &ln,
                                           int i, Acc<U32, DPL> &acc)
{
    const uint32_t d = chunk + i * desc_stride(DEPTH);
    // absolute address of the table (256-aligned: the buffer is 1024-aligned), so
    // leaf_addrs yields absolute leaf addresses with no base add
    const uint32_t tb = sabs(chunk + desc_bytes + i * table_stride(DEPTH));
    uint32_t a[DPL];
    leaf_addrs<DEPTH, DPL>(d, ln, tb, a);
    acc.add4(a);
}

// All NK trees of the warp in one unrolled block: ptxas schedules the whole chunk
// (descriptor, code-word and gather loads of every tree in flight together) instead
// of one loop iteration at a time (c3, 6 trees per warp: fused 6.37 -> 6.14 ms).
template <int DEPTH, bool U32, int DPL, int NK>
__device__ __forceinline__ void apply_trees_all(uint32_t chunk, uint32_t desc_bytes, const Lane &ln, int warp,
                                                Acc<U32, DPL> &acc)
{
#pragma unroll
    for (int k = 0; k < NK; ++k) apply_tree<DEPTH, U32, DPL>(chunk, desc_bytes, ln, warp + k * kConsumerWarps, acc);
}

template <int DEPTH, bool U32, int DPL = 4>
__device__ __forceinline__ void apply_chunk(uint32_t chunk, uint32_t desc_bytes, const Lane &ln,
                                            int warp, int nk, Acc<U32, DPL> &acc)
{
    // chunks hold nk * 16 trees (the last one padded with zero-answer trees).
    // (A software pipeline loading the next pair's descriptors during this pair was
    // slower: c3 fused 6.43 -> 7.66 ms.)
    // a multiple of 4 trees per warp runs 4 trees per iteration; 6 (c3's 96-tree
    // chunks) all at once.  (A switch fully unrolling 3..8 trees measured slower on
    // c3: 6.44 / 6.46 ms, larger code; so only these two shapes.)
    if (DEPTH <= 6 && (nk & 3) == 0) {
#pragma unroll 4
        for (int k = 0; k < nk; ++k) apply_tree<DEPTH, U32, DPL>(chunk, desc_bytes, ln, warp + k * kConsumerWarps, acc);
        return;
    }
    if (DEPTH <= 6 && nk == 6) {
        apply_trees_all<DEPTH, U32, DPL, 6>(chunk, desc_bytes, ln, warp, acc);
        return;
    }
#pragma unroll kApplyUnroll
    for (int k = 0; k < nk; ++k) apply_tree<DEPTH, U32, DPL>(chunk, desc_bytes, ln, warp + k * kConsumerWarps, acc);
}

// Fixed-order combine of the 16 group partials of document tid (< tile_docs) and store:
// score = (((P_0 + P_1) + P_2) + ... + P_15).
template <int DPL>
__device__ __forceinline__ void finish_doc(const KParams &p, uint32_t red, int tid, int64_t doc,
                                           int tile_docs, Acc<false, DPL> *)
{
    float s = lds_f32(red + tid * 4);
#pragma unroll
    for (int g = 1; g < kConsumerWarps; ++g) s += lds_f32(red + (g * tile_docs + tid) * 4);
    if (doc < p.n_docs) p.scores[doc] = s;
}
template <int DPL>
__device__ __forceinline__ void finish_doc(const KParams &p, uint32_t red, int tid, int64_t doc,
                                           int tile_docs, Acc<true, DPL> *)
{
    unsigned long long r = 0;
#pragma unroll
    for (int g = 0; g < kConsumerWarps; ++g) r += sld<unsigned long long>(red + (g * tile_docs + tid) * 8);
    if (doc < p.n_docs) {
        if (p.sums) p.sums[doc] = r;
        // (R - 2^31) * S + B, rounded op by op (no FMA contraction)
        if (p.dscores)
            p.dscores[doc] = __dadd_rn(__dmul_rn(__dsub_rn(static_cast<double>(r), 2147483648.0), p.scale),
                                       p.bias);
    }
}

// Split factors (> 127 borders) loaded as true bins: column A <- min(bin,127),
// column B <- max(bin-127, 0).
template <int DPL = 4>
__device__ __forceinline__ void expand_splits(const KParams &p, uint32_t bins, int tid, int nthr)
{
    constexpr int kT = 32 * DPL, CSH = DPL == 4 ? 0 : 1;  // tile documents, column shift
    for (int k = tid; k < p.n_split * (kT / 4); k += nthr) {
        const uint2 sp = p.splits[k / (kT / 4)];
        const uint32_t wd = (k % (kT / 4)) * 4, ca = sp.x >> CSH, cb = sp.y >> CSH;
        const uint32_t w = lds_u32(bins + ca + wd);
        sts_u32(bins + ca + wd, __vminu4(w, 0x7f7f7f7fu));
        sts_u32(bins + cb + wd, __vsubus4(w, 0x7f7f7f7fu));
    }
}

// Wide models (NEXT-4): u16 true bins of a tile (staged at `stage`, [n_used][128])
// -> every code column: column A <- min(bin, 127), B_c <- clamp(bin - 127c, 0, 127)
// (p.ucols[u] = {first B column * 128 or trash, C}).
__device__ __forceinline__ void expand_wide(const KParams &p, uint32_t stage, uint32_t codes, int tid,
                                            int nthr)
{
    for (int k = tid; k < p.n_used * (kTile / 4); k += nthr) {
        const int u = k / (kTile / 4);
        const uint32_t wd = (k % (kTile / 4)) * 4;  // first of the 4 documents
        const uint2 w = sld<uint2>(stage + 2u * (u * kTile + wd));  // 4 x u16
        const uint2 uc = p.ucols[u];
        sts_u32(codes + u * kTile + wd,
                prmt(__vminu2(w.x, 0x007f007fu), __vminu2(w.y, 0x007f007fu), 0x6420u));
        for (uint32_t c = 1; c < uc.y; ++c) {
            const uint32_t off = 127u * c * 0x00010001u;
            sts_u32(codes + uc.x + (c - 1u) * kTile + wd,
                    prmt(__vminu2(__vsubus2(w.x, off), 0x007f007fu),
                         __vminu2(__vsubus2(w.y, off), 0x007f007fu), 0x6420u));
        }
    }
}

// Phase A of one tile: the tile's factor jobs from the ring (slot / phase carried
// across phases and tiles).  A job's slot holds, per 32-factor sub-tile, H boxes of
// 128 documents (one per tile half), then the sub-tiles' fmeta, then their border
// arrays.  Warp w binarizes quad w >> 1 of every box for documents 64 * (w & 1) +
// lane (+ 32); the codes of half h go to the code block at h * half_stride.  Only
// the tile's hv halves that hold documents are loaded and binarized.
template <bool CODES, bool WIDE, bool FM, int H, class Sink, int DPL = 4, bool SPLIT2 = false>
__device__ __forceinline__ void phase_a(const KParams &p, const Sink sink, uint32_t ring, uint32_t bars,
                                        int n_fjobs, int S, int warp, int lane, uint32_t &slot,
                                        uint32_t &ph, unsigned long long &wait_ns, int hv)
{
    // 128-document tiles: warp w covers documents 64 (w & 1) + lane (+32); 64-document
    // tiles (DPL = 2): 32 (w & 1) + lane, code columns 64 bytes apart
    constexpr int NDL = DPL / 2, CSH = DPL == 4 ? 0 : 1;
    constexpr uint32_t kBox = 32u * DPL * kFSub * 4u;  // one TMA box: tile docs x 32 factors
    const int fsub = p.fsub_per_job, n_fchunks = p.n_fchunks;
    const uint32_t slot_bytes = p.slot_bytes, off_meta = p.off_meta, off_bord = p.off_bord,
                   bord_stride = p.bord_stride;
    // SPLIT2 (fused, 128-document tiles, one half; deep forests): warps 8h..8h+7
    // binarize the jobs j with j % 2 == h, warp w quad w & 7 for all 128 documents (4 per
    // lane): two jobs in progress at once and twice the work per job set-up; each warp
    // of the half arrives twice on the job's empty barrier (16 arrivals).  c4 (depth 10,
    // two-sub-tile jobs): fused 28.2 -> 26.4 ms; at depth 6 it costs more than it saves
    // (c3 6.14 -> 6.59 ms, c2 0.244 -> 0.250 ms), so only depth >= 7 uses it.
    if constexpr (SPLIT2 && CODES && H == 1 && DPL == 4) {
        const int q2 = warp & 7, half = warp >> 3;
        for (int j = 0; j < n_fjobs; ++j) {
            if ((j & 1) == half) {
                const uint32_t full = bars + 16u * slot, empty = full + 8u;
                mbar_wait(full, ph);
                const int nsub = min(fsub, n_fchunks - j * fsub);
                const uint32_t sb = ring + slot * slot_bytes;
                for (int s = 0; s < nsub; ++s)
                    binarize_sub<4, CODES, WIDE, FM, Sink, 0>(sb + s * kBox, sb + off_meta + s * kMetaBytes,
                                                             sb + off_bord + s * bord_stride, sink, q2, 0, lane);
                __syncwarp();
                if (lane == 0) mbar_arrive_cnt(empty, 2);
            }
            if (++slot == static_cast<uint32_t>(S)) {
                slot = 0;
                ph ^= 1u;
            }
        }
        (void)wait_ns;
        return;
    }
    const int q = warp >> 1, dbase = (warp & 1) * 32 * NDL;
    for (int j = 0; j < n_fjobs; ++j) {
        const uint32_t full = bars + 16u * slot, empty = full + 8u;
        DIAG_T(tw0);
        mbar_wait(full, ph);
#if ODF_DIAG & 8
        wait_ns += gtime() - tw0;
#else
        (void)wait_ns;
#endif
        const int nsub = min(fsub, n_fchunks - j * fsub);
        const uint32_t sb = ring + slot * slot_bytes;
#if ODF_DIAG & 1  // diagnostics build only: phase A does no work (TMA streaming rate)
        if (nsub < 0)
#endif
        for (int s = 0; s < nsub; ++s) {
            if constexpr (H == 1) {
                binarize_sub<NDL, CODES, WIDE, FM, Sink, CSH>(sb + s * kBox, sb + off_meta + s * kMetaBytes,
                                                            sb + off_bord + s * bord_stride, sink, q, dbase,
                                                            lane);
            } else {
                for (int h = 0; h < hv; ++h)
                    binarize_sub<2, CODES, WIDE, FM>(sb + (s * H + h) * kFSubBytes, sb + off_meta + s * kMetaBytes,
                                                     sb + off_bord + s * bord_stride, sink.at(h * p.half_stride),
                                                     q, dbase, lane);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty);
        if (++slot == static_cast<uint32_t>(S)) {
            slot = 0;
            ph ^= 1u;
        }
    }
}

// ---------------------------------------------------------------------------
// Main persistent kernel: MODE_FUSED (K3), MODE_BINARIZE (K1), MODE_APPLY (K2)
// WIDE: model with > 254 borders on some factor (NEXT-4): the wide search path in
// phase A, and u16 true bins from MODE_BINARIZE.
// H: tile halves.  A tile is H x 128 documents; each half has its own code block
// [n_cols + 1][128] (half_stride bytes apart), built from its own TMA box per
// factor sub-tile.  H = 2 (fused / apply, fp32 narrow models) lets one staged tree
// chunk serve 256 documents: half the L2 -> shared-memory forest traffic per
// document, which binds deep forests (c4: 16.6 MB of depth-10 tables per tile).
// Phase B with H = 2: warp w applies tree slot j = w & 7 of every half-chunk
// (tc / 2 trees, one ring slot) to half w >> 3.  A warp's trees are then t = j, j+8,
// j+16, ... of the forest, whose summation groups t mod 16 alternate j, j+8, j, ...,
// so two accumulators (swapped after every tree) keep the 16-group order of H = 1:
// scores are bit-identical for any H.
// ---------------------------------------------------------------------------
// halves of tile `tile` (H x 128 documents) that hold documents
template <int H>
__device__ __forceinline__ int valid_halves(int64_t n_docs, int64_t tile)
{
    if (H == 1) return 1;
    const int64_t v = (n_docs - tile * (kTile * H) + kTile - 1) / kTile;
    return v < H ? static_cast<int>(v) : H;
}

template <int MODE, int DEPTH, bool U32, bool WIDE, int H = 1, int DPL = 4>
__global__ void __launch_bounds__(kThreads, MODE == MODE_BINARIZE ? 2 : 1)  // K1: 2 CTAs per SM
    odf_main_kernel(const KParams p, const __grid_constant__ CUtensorMap tmap)
{
    constexpr bool HAS_A = MODE != MODE_APPLY;
    constexpr bool HAS_B = MODE != MODE_BINARIZE;
    constexpr int kT = 32 * DPL;                 // documents per tile half (128, or 64 for wide-column models)
    constexpr uint32_t kBox = kT * kFSub * 4u;   // one TMA box: kT docs x 32 factors
    constexpr int kTileH = kT * H;               // documents per tile
    constexpr int kSlots = kConsumerWarps / H;   // tree slots per half (phase B)
    constexpr bool MIXED = DEPTH == kMixedDepth;  // per-segment depths (NEXT-2)
    static_assert(!MIXED || (H == 1 && U32), "mixed-height models: integer answers, 128-doc tiles");
    static_assert(DPL == 4 || (DPL == 2 && H == 1 && !WIDE), "64-document tiles: narrow models, one half");
    static_assert(H == 1 || (H == 2 && !WIDE && MODE != MODE_BINARIZE), "halves: fused/apply, narrow");
    if (smem_addr(smem_raw) & 1023u) __trap();  // alignment the TMA swizzle relies on
    const uint32_t base = 0;
    const uint32_t bins = base + p.off_bins;
    const uint32_t ring = base + p.off_ring;
    const uint32_t red = base + p.off_red;
    const uint32_t bars = base + p.off_bars;
    const int S = p.stages;
    // bars: [0,128) full/empty of up to 8 stages, [128,144) bins_full/empty,
    // [144,160) scratch word for Acc::pin, [160,...) copy of p.bchunk
    const uint32_t bins_full = bars + 128u, bins_empty = bins_full + 8u;
    const uint32_t pin_scratch = bars + 144u;
    const uint32_t bct = bars + 160u;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_fjobs = HAS_A ? (p.n_fchunks + p.fsub_per_job - 1) / p.fsub_per_job : 0;
    // ring jobs of phase B: tree chunks (H = 1) or half-chunks of tc / 2 trees (H = 2)
    const int n_bjobs = HAS_B && !MIXED ? p.n_tchunks * H : 0;
    constexpr bool WIDE_BINS = MODE == MODE_BINARIZE && WIDE;
    const uint32_t tile_bins_bytes = static_cast<uint32_t>(p.n_used) * kT * (p.wide ? 2u : 1u);
    const uint32_t bins_dst = (MODE == MODE_APPLY && p.wide) ? base + p.off_stage : bins;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(bars + 16u * s, 1);                   // full[s]: producer + tx bytes
            mbar_init(bars + 16u * s + 8u, kConsumerWarps);  // empty[s]: one arrive per warp
        }
        mbar_init(bins_full, 1);
        mbar_init(bins_empty, kConsumerWarps);
        fence_barrier_init();
    }
    if (HAS_A)
        for (int c = threadIdx.x; c < p.n_fchunks; c += kThreads) sst<uint2>(bct + 8u * c, p.bchunk[c]);
    __syncthreads();
    // partly filled last wave (odf_score_tiles): the 64-document-tile secondary launch may
    // start as soon as SMs free up
    if (p.pdl == 1 && threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (warp == kConsumerWarps) {
        // ===================== producer warp (one elected lane) =====================
        if (lane == 0) {
            if (HAS_A && n_fjobs > 0)
                asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap))
                             : "memory");
            uint32_t slot = 0, ph = 0, bph = 0;
            for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
                // halves holding documents (a fully out-of-range half is not loaded)
                const int hv = valid_halves<H>(p.n_docs, tile);
                if (MODE == MODE_APPLY && tile_bins_bytes > 0) {
                    mbar_wait(bins_empty, bph ^ 1u);
                    mbar_expect_tx(bins_full, tile_bins_bytes * hv);
                    for (int h = 0; h < hv; ++h)
                        bulk_g2s(bins_dst + h * p.half_stride, p.bins_in + (tile * H + h) * tile_bins_bytes,
                                 tile_bins_bytes, bins_full);
                    bph ^= 1u;
                }
                for (int j = 0; j < n_fjobs; ++j) {
                    const uint32_t full = bars + 16u * slot, empty = full + 8u;
                    mbar_wait(empty, ph ^ 1u);
                    const int c0 = j * p.fsub_per_job;
                    const int nsub = min(p.fsub_per_job, p.n_fchunks - c0);
                    const uint32_t sb = ring + slot * p.slot_bytes;
                    uint32_t tx = 0;
                    for (int s = 0; s < nsub; ++s)
                        tx += kBox * hv + kMetaBytes + sld<uint2>(bct + 8u * (c0 + s)).y;
                    mbar_expect_tx(full, tx);
                    for (int s = 0; s < nsub; ++s) {
                        const int c = c0 + s;
                        for (int h = 0; h < hv; ++h) {
                            const int row = static_cast<int>(tile * kTileH + h * kT);
                            if (p.fm)  // feature-major input (NEXT-4): box (kT docs, 32 factors)
                                tma_load_2d(sb + (s * H + h) * kBox, &tmap, row, c * kFSub, full);
                            else
                                tma_load_2d(sb + (s * H + h) * kBox, &tmap, c * kFSub, row, full);
                        }
                        bulk_g2s(sb + p.off_meta + s * kMetaBytes, p.fmeta + c * kFSub, kMetaBytes,
                                 full);
                        const uint2 bc = sld<uint2>(bct + 8u * c);
                        if (bc.y)
                            bulk_g2s(sb + p.off_bord + s * p.bord_stride,
                                     reinterpret_cast<const char *>(p.borders) + bc.x, bc.y, full);
                    }
                    if (++slot == static_cast<uint32_t>(S)) { slot = 0; ph ^= 1u; }
                }
                if constexpr (MIXED) {  // every segment's chunks, in segment order
                    for (int sg = 0; sg < p.n_seg; ++sg)
                        for (int c = 0; c < p.seg[sg].n_chunks; ++c) {
                            const uint32_t full = bars + 16u * slot, empty = full + 8u;
                            mbar_wait(empty, ph ^ 1u);
                            const uint32_t cb = p.seg[sg].chunk_bytes;
                            mbar_expect_tx(full, cb);
                            bulk_g2s(ring + slot * p.slot_bytes,
                                     p.chunks + p.seg[sg].byte_off + static_cast<size_t>(c) * cb, cb, full);
                            if (++slot == static_cast<uint32_t>(S)) { slot = 0; ph ^= 1u; }
                        }
                }
                for (int c = 0; c < n_bjobs; ++c) {
                    const uint32_t full = bars + 16u * slot, empty = full + 8u;
                    mbar_wait(empty, ph ^ 1u);
                    const uint32_t sb = ring + slot * p.slot_bytes;
                    if constexpr (H == 1) {
                        mbar_expect_tx(full, p.chunk_bytes);
                        bulk_g2s(sb, p.chunks + static_cast<size_t>(c) * p.chunk_bytes, p.chunk_bytes, full);
                    } else {
                        // half-chunk q of chunk c >> 1: its descriptors, then its tables at hdesc_bytes
                        const int half_tc = p.tc / 2;
                        const uint8_t *ch = p.chunks + static_cast<size_t>(c >> 1) * p.chunk_bytes;
                        const uint32_t db = static_cast<uint32_t>(half_tc * desc_stride(DEPTH));
                        const uint32_t tbytes = static_cast<uint32_t>(half_tc * table_stride(DEPTH));
                        mbar_expect_tx(full, db + tbytes);
                        bulk_g2s(sb, ch + (c & 1) * db, db, full);
                        bulk_g2s(sb + p.hdesc_bytes, ch + p.desc_bytes + (c & 1) * tbytes, tbytes, full);
                    }
                    if (++slot == static_cast<uint32_t>(S)) { slot = 0; ph ^= 1u; }
                }
            }
        }
        return;
    }

    // ========================= consumer warps =========================
    const int tid = threadIdx.x;
    const int half = H == 1 ? 0 : warp / kSlots, tslot = H == 1 ? warp : warp % kSlots;
    const Lane ln = make_lane(p, sabs(bins + half * p.half_stride) + lane * DPL);  // absolute (tree_flags)
    const uint32_t desc_off = H == 1 ? p.desc_bytes : p.hdesc_bytes;  // tables in a ring slot
    const int nk = H == 1 ? p.tc / kConsumerWarps : p.tc / (2 * kSlots);  // trees per job per warp
    uint32_t slot = 0, ph = 0, bph = 0;
#if ODF_DIAG & 8
    int diag_it = 0;
#endif
    for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const int hv = valid_halves<H>(p.n_docs, tile);
        unsigned long long waitA = 0;
#if ODF_DIAG & 8
        unsigned long long waitB = 0;
#endif
        DIAG_T(t_start);
        if constexpr (MODE == MODE_BINARIZE) {  // K1: bins straight to HBM, no shared-memory tile
            const uint32_t lim = static_cast<uint32_t>(p.n_used) * kT;
            if constexpr (WIDE_BINS) {
                const GmemBinsSink16 snk{reinterpret_cast<uint16_t *>(p.bins_out + tile * tile_bins_bytes), lim};
                if (p.fm)
                    phase_a<false, true, true, 1>(p, snk, ring, bars, n_fjobs, S, warp, lane, slot, ph, waitA, hv);
                else
                    phase_a<false, true, false, 1>(p, snk, ring, bars, n_fjobs, S, warp, lane, slot, ph, waitA, hv);
            } else {
                const GmemBinsSink snk{p.bins_out + tile * tile_bins_bytes, lim};
                if (p.fm)
                    phase_a<false, false, true, 1, GmemBinsSink, DPL>(p, snk, ring, bars, n_fjobs, S, warp, lane,
                                                                      slot, ph, waitA, hv);
                else
                    phase_a<false, false, false, 1, GmemBinsSink, DPL>(p, snk, ring, bars, n_fjobs, S, warp, lane,
                                                                       slot, ph, waitA, hv);
            }
            continue;
        } else if (HAS_A) {
            {
                if (p.fm)
                    phase_a<MODE == MODE_FUSED, WIDE, true, H, SmemSink, DPL, (DEPTH >= ODF_SPLIT_MIN_DEPTH && !MIXED)>(p, SmemSink{bins}, ring, bars, n_fjobs,
                                                                              S, warp, lane, slot, ph, waitA, hv);
                else
                    phase_a<MODE == MODE_FUSED, WIDE, false, H, SmemSink, DPL, (DEPTH >= ODF_SPLIT_MIN_DEPTH && !MIXED)>(p, SmemSink{bins}, ring, bars, n_fjobs,
                                                                               S, warp, lane, slot, ph, waitA, hv);
            }
        }
        if (MODE == MODE_APPLY && tile_bins_bytes > 0) {
            mbar_wait(bins_full, bph);
            bph ^= 1u;
            if (p.wide)
                expand_wide(p, base + p.off_stage, bins, tid, kConsumerThreads);
            else
                for (int h = 0; h < hv; ++h) expand_splits<DPL>(p, bins + h * p.half_stride, tid, kConsumerThreads);
        }
        DIAG_T(t_adone);
        named_bar_consumers();  // all bins of the tile written
        DIAG_T(t_bstart);

        // acc: the group of the warp's next tree; acc2 (H = 2): the other group
        Acc<U32, DPL> acc, acc2;
        if constexpr (MIXED) {
            for (int sg = 0; sg < p.n_seg; ++sg) {
                const int sd = p.seg[sg].depth, snk = p.seg[sg].tc / kConsumerWarps;
                const uint32_t sdesc = p.seg[sg].desc_bytes;
                for (int c = 0; c < p.seg[sg].n_chunks; ++c) {
                    const uint32_t full = bars + 16u * slot, empty = full + 8u;
                    mbar_wait(full, ph);
                    const uint32_t sb = ring + slot * p.slot_bytes;
                    switch (sd) {  // warp-uniform: one branch per chunk
                        case 0: apply_chunk<0, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 1: apply_chunk<1, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 2: apply_chunk<2, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 3: apply_chunk<3, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 4: apply_chunk<4, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 5: apply_chunk<5, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 6: apply_chunk<6, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 7: apply_chunk<7, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 8: apply_chunk<8, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        case 9: apply_chunk<9, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                        default: apply_chunk<10, U32, DPL>(sb, sdesc, ln, tslot, snk, acc); break;
                    }
                    acc.pin(pin_scratch);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty);
                    if (++slot == static_cast<uint32_t>(S)) { slot = 0; ph ^= 1u; }
                }
            }
        }
        for (int c = 0; c < n_bjobs; ++c) {
            const uint32_t full = bars + 16u * slot, empty = full + 8u;
            DIAG_T(tw0);
            mbar_wait(full, ph);
#if ODF_DIAG & 8
            waitB += gtime() - tw0;
#endif
            const uint32_t sb = ring + slot * p.slot_bytes;
#if ODF_DIAG & 2  // diagnostics build only: phase B does no work
            if (n_bjobs < 0)
#endif
            {
                if constexpr (MIXED) {
                } else if constexpr (H == 1) {
                    apply_chunk<DEPTH, U32, DPL>(sb, desc_off, ln, tslot, nk, acc);
                } else {
#pragma unroll 2
                    for (int k = 0; k < nk; ++k) {
                        apply_tree<DEPTH, U32, DPL>(sb, desc_off, ln, tslot + k * kSlots, acc);
                        const Acc<U32, DPL> t = acc;
                        acc = acc2;
                        acc2 = t;
                    }
                }
            }
            acc.pin(pin_scratch);
            if (H > 1) acc2.pin(pin_scratch);
            __syncwarp();
            if (lane == 0) mbar_arrive(empty);
            if (++slot == static_cast<uint32_t>(S)) { slot = 0; ph ^= 1u; }
        }
        DIAG_T(t_bdone);
        // reduction buffer aliases the bins: wait until every warp is done with them
        named_bar_consumers();
        // a warp applies an even number of trees per tile (tc is a multiple of 16), so
        // acc holds group tslot and acc2 group tslot + 8 (H = 2)
        acc.to_red(red, tslot, half * kT + lane * DPL, kTileH);
        if (H > 1) acc2.to_red(red, tslot + kSlots, half * kT + lane * DPL, kTileH);
        named_bar_consumers();
        if (tid < kTileH)
            finish_doc(p, red, tid, tile * kTileH + tid, kTileH, static_cast<Acc<U32, DPL> *>(nullptr));
        if (MODE == MODE_APPLY && tile_bins_bytes > 0) {
            fence_proxy_async();  // generic writes to the bins region precede the next TMA
        }
        named_bar_consumers();
        if (MODE == MODE_APPLY && tile_bins_bytes > 0 && lane == 0) mbar_arrive(bins_empty);
#if ODF_DIAG & 8
        if (lane == 0 && diag_it < kDiagIt && blockIdx.x < 148) {
            unsigned long long *d = g_diag + ((static_cast<size_t>(blockIdx.x) * kDiagIt + diag_it) * 16 + warp) * 8;
            d[0] = t_start; d[1] = t_adone; d[2] = t_bstart; d[3] = t_bdone; d[4] = gtime();
            d[5] = waitA; d[6] = waitB; d[7] = static_cast<unsigned long long>(tile);
        }
        ++diag_it;
#endif
    }
    // secondary of a programmatic dependent launch: complete only after the primary, so
    // later stream work sees both grids' scores
    if (p.pdl == 2) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------------------
// K6: leaf-index export and per-document fingerprint (tests).  Same tree_flags
// as the apply path; bins and descriptors staged in shared memory by plain loads.
// ---------------------------------------------------------------------------
template <int DEPTH, int DPL = 4>
__global__ void __launch_bounds__(kConsumerThreads)
    odf_index_kernel(const KParams p, int fingerprint)
{
    constexpr int kT = 32 * DPL;  // documents per tile
    if (smem_addr(smem_raw) & 1023u) __trap();
    const uint32_t base = 0;
    const uint32_t bins = base;
    const uint32_t descs = base + ((static_cast<uint32_t>(p.n_cols) * kT + 1023u) & ~1023u);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t tile_bins_bytes = static_cast<uint32_t>(p.n_used) * kT * (p.wide ? 2u : 1u);
    const int64_t tile = (fingerprint ? 0 : p.doc0 / kT) + blockIdx.x;
    {
        const uint32_t dst = p.wide ? p.off_stage : bins;
        const uint4 *src = reinterpret_cast<const uint4 *>(p.bins_in + tile * tile_bins_bytes);
        for (uint32_t k = tid; k < tile_bins_bytes / 16; k += kConsumerThreads)
            sts_v4u(dst + 16 * k, __ldg(src + k));
        __syncthreads();
        if (p.wide)
            expand_wide(p, p.off_stage, bins, tid, kConsumerThreads);
        else
            expand_splits<DPL>(p, bins, tid, kConsumerThreads);
        __syncthreads();
    }
    const Lane ln = make_lane(p, sabs(bins) + lane * DPL);  // absolute (tree_flags)
    const int64_t t_lo = fingerprint ? 0 : p.tree0;
    const int64_t t_hi = fingerprint ? p.n_trees : p.tree0 + p.ntree;
    uint64_t h[DPL];
#pragma unroll
    for (int n = 0; n < DPL; ++n) h[n] = 0xcbf29ce484222325ull;
    for (int64_t c = t_lo / p.tc; c * p.tc < t_hi; ++c) {
        const uint8_t *chunk = p.chunks + static_cast<size_t>(c) * p.chunk_bytes;
        const uint32_t dbytes = static_cast<uint32_t>(p.tc) * desc_stride(DEPTH);
        for (uint32_t k = tid; k < dbytes / 16; k += kConsumerThreads)
            sts_v4u(descs + 16 * k, __ldg(reinterpret_cast<const uint4 *>(chunk) + k));
        __syncthreads();
        const int64_t c0 = c * p.tc;
        if (fingerprint) {
            if (warp == 0) {
                for (int i = 0; i < p.tc && c0 + i < p.n_trees; ++i) {
                    uint32_t F[DPL];
                    tree_findex<DEPTH, DPL>(descs + i * desc_stride(DEPTH), ln, F);
#pragma unroll
                    for (int n = 0; n < DPL; ++n) {
                        const uint32_t idx = F[n] ^ ((1u << DEPTH) - 1u);
                        h[n] = (h[n] ^ (idx & 0xffu)) * 0x100000001b3ull;
                        h[n] = (h[n] ^ (idx >> 8)) * 0x100000001b3ull;
                    }
                }
            }
        } else {
            for (int i = warp; i < p.tc; i += kConsumerWarps) {
                const int64_t t = c0 + i;
                if (t < p.tree0 || t >= t_hi) continue;
                uint32_t F[DPL];
                tree_findex<DEPTH, DPL>(descs + i * desc_stride(DEPTH), ln, F);
#pragma unroll
                for (int n = 0; n < DPL; ++n) {
                    const int64_t doc = tile * kT + lane * DPL + n;
                    if (doc >= p.doc0 && doc < p.doc0 + p.ndoc)
                        p.idx_out[(doc - p.doc0) * p.ntree + (t - p.tree0)] =
                            static_cast<uint16_t>(F[n] ^ ((1u << DEPTH) - 1u));
                }
            }
        }
        __syncthreads();
    }
    if (fingerprint && warp == 0) {
#pragma unroll
        for (int n = 0; n < DPL; ++n) {
            const int64_t doc = tile * kT + lane * DPL + n;
            if (doc < p.n_docs) p.fp_out[doc] = h[n];
        }
    }
}

// ---------------------------------------------------------------------------
// K4: small-batch latency path (config c5).  Two launches:
//  (1) odf_lat_binarize_kernel, grid (n_fchunks, n_tiles): one CTA per 128-doc x
//      32-factor sub-tile writes its 7-bit code columns to a global [tile][n_cols][128]
//      block (L2-resident), so binarization of one tile is spread over many SMs;
//  (2) odf_lat_apply_kernel, grid (S, n_tiles): CTA s applies the tree chunks
//      [s*C/S, (s+1)*C/S) to its tile and writes a partial [128]; the last CTA of
//      a tile (atomic ticket) sums the S partials in ascending s -> deterministic.
// The association differs from the main path (tree ranges per split), so these
// scores are held to the tolerance, not bit-exactness.
// ---------------------------------------------------------------------------
// DPL: documents per lane of the model's tiles (4: 128-document tiles; 2: 64-document
// tiles of wide-column models, whose column offsets are halved, CSH = 1)
template <int DPL>
__global__ void __launch_bounds__(kConsumerThreads)
    odf_lat_binarize_kernel(const KParams p, const __grid_constant__ CUtensorMap tmap)
{
    constexpr int kT = 32 * DPL, NDL = DPL / 2, CSH = DPL == 4 ? 0 : 1;
    constexpr uint32_t kBox = kT * kFSub * 4u;  // one TMA box: kT docs x 32 factors
    if (smem_addr(smem_raw) & 1023u) __trap();
    const int c = blockIdx.x;
    const int64_t tile = blockIdx.y;
    const uint32_t t_off = 0, m_off = kBox, b_off = kBox + kMetaBytes;
    const uint32_t bar = b_off + ((p.bord_stride + 15u) & ~15u);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
        const uint2 bc = p.bchunk[c];
        mbar_expect_tx(bar, kBox + kMetaBytes + bc.y);
        if (p.fm)
            tma_load_2d(t_off, &tmap, static_cast<int>(tile * kT), c * kFSub, bar);
        else
            tma_load_2d(t_off, &tmap, c * kFSub, static_cast<int>(tile * kT), bar);
        bulk_g2s(m_off, p.fmeta + c * kFSub, kMetaBytes, bar);
        if (bc.y) bulk_g2s(b_off, reinterpret_cast<const char *>(p.borders) + bc.x, bc.y, bar);
        if (c == 0) p.lat_counter[tile] = 0u;  // ticket for kernel (2), stream-ordered
    }
    // programmatic dependent launch: kernel (2) may start now (it stages its first
    // tree chunk, then waits for this grid with griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __syncthreads();
    mbar_wait(bar, 0);
    const GmemSink sink{p.lat_codes + tile * p.code_stride};
    constexpr bool WIDE = DPL == 4;  // > 254-border factors: 128-document models only
    if (p.fm)
        binarize_sub<NDL, true, WIDE, true, GmemSink, CSH>(t_off, m_off, b_off, sink, warp >> 1,
                                                           (warp & 1) * 32 * NDL, lane);
    else
        binarize_sub<NDL, true, WIDE, false, GmemSink, CSH>(t_off, m_off, b_off, sink, warp >> 1,
                                                            (warp & 1) * 32 * NDL, lane);
}

// U32: integer leaves (NEXT-1), u64 partials per split summed exactly (order-free: the
// result equals odf_score_u64 bit for bit); DEPTH == kMixedDepth: height segments
// (NEXT-2), each chunk applied at its segment's depth.
template <int DEPTH, int DPL = 4, bool U32 = false>
__global__ void __launch_bounds__(kConsumerThreads)
    odf_lat_apply_kernel(const KParams p)
{
    constexpr int kT = 32 * DPL;  // documents per tile
    constexpr bool MIXED = DEPTH == kMixedDepth;
    static_assert(!MIXED || U32, "mixed-height models: integer answers");
    if (smem_addr(smem_raw) & 1023u) __trap();
    const int split = blockIdx.x, S = gridDim.x;
    const int64_t tile = blockIdx.y;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // shared memory: the tile's code columns, p.stages (1 or 2) tree-chunk buffers, the
    // reduction buffer, mbarriers [codes, chunk buffer 0, chunk buffer 1]; everything is
    // staged with bulk copies (cp.async.bulk), not thread loops
    const uint32_t bins = 0;
    const uint32_t cols_bytes = static_cast<uint32_t>(p.n_cols) * kT;
    const uint32_t chunk_al = (p.chunk_bytes + 1023u) & ~1023u;
    const uint32_t chunk0 = (cols_bytes + 1023u) & ~1023u;
    const int nbuf = p.stages;
    const uint32_t red = chunk0 + nbuf * chunk_al;
    const uint32_t bar = red + Acc<U32, DPL>::kRed;
    const int c_lo = static_cast<int>(static_cast<int64_t>(split) * p.n_tchunks / S);
    const int c_hi = static_cast<int>(static_cast<int64_t>(split + 1) * p.n_tchunks / S);
    // chunk c of the stream: its segment (mixed-height models; one segment otherwise)
    auto seg_of = [&](int c) {
        int sg = 0;
        if constexpr (MIXED)
            while (sg + 1 < p.n_seg && c >= p.seg[sg].n_chunks) c -= p.seg[sg++].n_chunks;
        return make_int2(sg, c);
    };
    auto stage_chunk = [&](int c, int b) {  // one thread
        uint32_t cb = p.chunk_bytes;
        const uint8_t *src = p.chunks + static_cast<size_t>(c) * p.chunk_bytes;
        if constexpr (MIXED) {
            const int2 sc = seg_of(c);
            cb = p.seg[sc.x].chunk_bytes;
            src = p.chunks + p.seg[sc.x].byte_off + static_cast<size_t>(sc.y) * cb;
        }
        mbar_expect_tx(bar + 8u + 8u * b, cb);
        bulk_g2s(chunk0 + b * chunk_al, src, cb, bar + 8u + 8u * b);
    };
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 8u, 1);
        mbar_init(bar + 16u, 1);
        fence_barrier_init();
        // tree chunks do not depend on kernel (1): start them before waiting for that
        // grid (programmatic dependent launch; after a plain launch the wait is a no-op)
        for (int b = 0; b < nbuf && c_lo + b < c_hi; ++b) stage_chunk(c_lo + b, b);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0 && cols_bytes > 0) {  // the codes kernel (1) wrote, now complete and visible
        mbar_expect_tx(bar, cols_bytes);
        bulk_g2s(bins, p.lat_codes + tile * p.code_stride, cols_bytes, bar);
    }
    __syncthreads();  // barrier initialisation visible to every thread
    if (cols_bytes > 0) mbar_wait(bar, 0);
    Acc<U32, DPL> acc;
    const Lane ln = make_lane(p, sabs(bins) + lane * DPL);  // absolute (tree_flags)
    uint32_t ph0 = 0, ph1 = 0;
    for (int c = c_lo, i = 0; c < c_hi; ++c, ++i) {
        const int b = nbuf == 2 ? (i & 1) : 0;
        mbar_wait(bar + 8u + 8u * b, b ? ph1 : ph0);
        if (b) ph1 ^= 1u; else ph0 ^= 1u;
        const uint32_t cb = chunk0 + b * chunk_al;
        if constexpr (MIXED) {
            const SegP &g = p.seg[seg_of(c).x];
            const int nk = g.tc / kConsumerWarps;
            switch (g.depth) {  // warp-uniform: one branch per chunk
                case 0: apply_chunk<0, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 1: apply_chunk<1, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 2: apply_chunk<2, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 3: apply_chunk<3, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 4: apply_chunk<4, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 5: apply_chunk<5, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 6: apply_chunk<6, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 7: apply_chunk<7, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 8: apply_chunk<8, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                case 9: apply_chunk<9, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
                default: apply_chunk<10, true, DPL>(cb, g.desc_bytes, ln, warp, nk, acc); break;
            }
        } else {
            apply_chunk<DEPTH, U32, DPL>(cb, p.desc_bytes, ln, warp, p.tc / kConsumerWarps, acc);
        }
        if (c + nbuf < c_hi) {  // refill buffer b once every warp's gathers from it are done
            acc.pin(bar + 24u);
            __syncthreads();
            if (tid == 0) stage_chunk(c + nbuf, b);
        }
    }
    acc.to_red(red, warp, lane * DPL, kT);
    __syncthreads();
    using Part = typename std::conditional<U32, unsigned long long, float>::type;
    Part *part = reinterpret_cast<Part *>(p.lat_partial) + (tile * S) * kT;
    if (tid < kT) {
        Part v = sld<Part>(red + tid * sizeof(Part));
#pragma unroll
        for (int w = 1; w < kConsumerWarps; ++w) v += sld<Part>(red + (w * kT + tid) * sizeof(Part));
        part[split * kT + tid] = v;
    }
    __threadfence();
    __syncthreads();
    __shared__ uint32_t last;
    if (tid == 0) last = (atomicAdd(p.lat_counter + tile, 1u) == static_cast<uint32_t>(S - 1)) ? 1u : 0u;
    __syncthreads();
    if (last && tid < kT) {
        __threadfence();
        Part v = __ldcg(part + tid);
        for (int s2 = 1; s2 < S; ++s2) v += __ldcg(part + s2 * kT + tid);
        const int64_t doc = tile * kT + tid;
        if (doc < p.n_docs) {
            if constexpr (U32) {
                if (p.sums) p.sums[doc] = v;
                // (R - 2^31) * S + B, rounded op by op (no FMA contraction)
                if (p.dscores)
                    p.dscores[doc] = __dadd_rn(
                        __dmul_rn(__dsub_rn(static_cast<double>(v), 2147483648.0), p.scale), p.bias);
            } else {
                p.scores[doc] = v;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// NEXT-3: bit-packed ordered condition words (the paper's "ordered format",
// §5.4: bit i <-> document i), one u32 per binary feature per 32
// documents, built with __ballot_sync; and an apply that assembles each leaf index
// from those words (§6.4).  Binary feature kb = (used factor u, border j),
// numbered by ascending u then j; its bit for document i is (bin(x_i) <= j), i.e.
// the node condition x < b_j itself.  Words: [ceil(D/32)][K_bin].
// ---------------------------------------------------------------------------
#ifdef ODF_KERNELS_AUX  // non-template kernels: defined in odf_k_aux.cu only
__global__ void __launch_bounds__(kConsumerThreads)
    odf_bits_from_bins_kernel(const KParams p)
{
    const int64_t tile = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kT = p.tile_docs;  // the model's bins tile width (128, or 64)
    const uint8_t *bt = p.bins_in + tile * static_cast<int64_t>(p.n_used) * kT * (p.wide ? 2 : 1);
    const uint16_t *bt16 = reinterpret_cast<const uint16_t *>(bt);
    for (int u = warp; u < p.n_used; u += kConsumerWarps) {
        const uint32_t base = p.bf_base[u], m = p.bf_base[u + 1] - base;
#pragma unroll 1
        for (int q = 0; q < kT / 32; ++q) {
            const int64_t g = tile * (kT / 32) + q;  // 32-document group
            if (g * 32 >= p.n_docs) break;
            const bool valid = g * 32 + lane < p.n_docs;  // padding documents: bit 0
            const uint32_t b = !valid ? 0xffffffffu
                               : p.wide ? bt16[u * kT + q * 32 + lane]
                                        : bt[u * kT + q * 32 + lane];
            uint32_t *dst = p.words + g * p.k_bin + base;
            for (uint32_t j0 = 0; j0 < m; j0 += 32) {
                uint32_t mine = 0;
                const uint32_t nj = min(32u, m - j0);
                for (uint32_t jj = 0; jj < nj; ++jj) {
                    const uint32_t w = __ballot_sync(0xffffffffu, b <= j0 + jj);
                    if (lane == static_cast<int>(jj)) mine = w;
                }
                if (static_cast<uint32_t>(lane) < nj) dst[j0 + lane] = mine;
            }
        }
    }
}
#endif

// One CTA per 32-document group; lane = document; warp w sums trees t = w mod 16 in
// ascending order and the 16 partials are combined in order: the same summation
// order as the main path, so scores are bit-identical to odf_score.
template <int DEPTH>
__global__ void __launch_bounds__(kConsumerThreads)
    odf_apply_bits_kernel(const KParams p)
{
    const int64_t g = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t *wg = p.words + g * p.k_bin;
    for (int64_t k = tid; k < p.k_bin; k += kConsumerThreads) sst<uint32_t>(4u * k, wg[k]);
    __syncthreads();
    const uint32_t red = (4u * static_cast<uint32_t>(p.k_bin) + 15u) & ~15u;
    float acc = 0.f;
    for (int64_t t = warp; t < p.n_trees; t += kConsumerWarps) {
        uint32_t idx = 0;
#pragma unroll
        for (int l = 0; l < DEPTH; ++l) {
            const uint32_t w = lds_u32(__ldg(p.bits_desc + t * DEPTH + l));  // broadcast
            idx |= ((w >> lane) & 1u) << l;
        }
        acc += __ldg(p.leaves + (t << DEPTH) + idx);
    }
    sst<float>(red + 4u * (warp * 32 + lane), acc);
    __syncthreads();
    if (tid < 32) {
        float s = lds_f32(red + 4u * tid);
#pragma unroll
        for (int w = 1; w < kConsumerWarps; ++w) s += lds_f32(red + 4u * (w * 32 + tid));
        const int64_t doc = g * 32 + tid;
        if (doc < p.n_docs) p.scores[doc] = s;
    }
}

}  // namespace odf
