// sa_search_staged.cuh -- long reads (m > 128 bases) with the phase-B verification staged in shared
// memory by TMA bulk copies (north_star: "staged in shared memory via TMA"; "warp-cooperative ...
// using __shfl/__ballot for suffix comparison").  Same result as k_match<0> (sa_search.cuh: the search
// of Alg. 1, corrected per DESIGN.md A4-A8, in two phases):
//
//  (A) per thread, the search for P' = P's first mt = k + (record-cached bases) bases: the records
//      decide every probe.  Its interval [lo', hi') holds P's interval (P' is a prefix of P).
//  (B) hi' - lo' == 1 (a unique P'; every exact long read of a non-repeat locus): ONE compare decides
//      P's interval, of P's bases [mt, m) against the suffix s = SA[lo'] from base mt.  s is the
//      split pivot of (A) (the only suffix with prefix P'), so its record was loaded there: no probe.
//      The warp collects its lanes' verifications in rounds of up to `slots`; in a round every
//      selected lane issues two cp.async.bulk copies (global -> shared, completing on the warp's
//      mbarrier): its read's bases [mt, m) and the text window at s + mt, 16-byte aligned word
//      ranges.  All windows of the round are in flight together (no registers held, unlike a load
//      chain), then the warp compares each window pair with lane j on word j (32 bases) and one
//      ballot finds the first difference (1024 bases per step).
//      hi' - lo' > 1 (a repeat longer than mt): the joint search of k_match<0> over [lo', hi').
//
// Result for the unique case (the joint search over (lo'-1, lo'+1) makes exactly this one probe):
//   P a prefix of t_s  -> [lo', lo'+1);   P < t_s -> [lo', lo');   P > t_s -> [lo'+1, lo'+1).
#pragma once

#include "sa_search.cuh"

namespace sa_search {

// The staged word range of a window of L >= 1 bases at absolute base b of a 2-bit stream: words
// [a0, a0 + words), a0 even (16-byte aligned when the stream is), through word (b+L-1)/32 + 1 (the
// funnel shift's next word), `words` even.  Window word j = (d[off+j] << sh) | (d[off+j+1] >> (64-sh)).
struct StageWin {
    uint64_t a0;
    uint32_t words;
    uint32_t off;
    uint32_t sh;
};

__device__ __forceinline__ StageWin stage_win(uint64_t b, uint32_t L) {
    const uint64_t w0 = b >> 5, w1 = (b + L - 1) >> 5;
    StageWin g;
    g.a0 = w0 & ~1ull;
    g.words = (uint32_t)(((w1 + 2) & ~1ull) - g.a0);
    g.off = (uint32_t)(w0 - g.a0);
    g.sh = (uint32_t)(b & 31u) << 1;
    return g;
}

// bytes the bulk copy of g moves from a stream of `total` readable words (the part below total & ~1)
__device__ __forceinline__ uint32_t stage_bulk_bytes(const StageWin &g, uint64_t total) {
    const uint64_t end = g.a0 + g.words, te = total & ~1ull, cend = end < te ? end : te;
    return cend > g.a0 ? (uint32_t)((cend - g.a0) * 8) : 0u;
}

// Issue the copy of g into dst (shared): one cp.async.bulk for the 16-byte-aligned part inside the
// stream, completing on the mbarrier `bar`; a trailing odd word by a plain load, zeros past the stream.
__device__ __forceinline__ void stage_issue(uint64_t *dst, const uint64_t *__restrict__ src, uint64_t total,
                                            const StageWin &g, uint32_t bar) {
    const uint32_t bytes = stage_bulk_bytes(g, total);
    if (bytes) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(d), "l"(src + g.a0), "r"(bytes), "r"(bar) : "memory");
    }
    for (uint32_t w = bytes / 8; w < g.words; ++w) dst[w] = g.a0 + w < total ? ld_u64(src + g.a0 + w) : 0ull;
}

__device__ __forceinline__ uint64_t stage_word(const uint64_t *d, uint32_t i, uint32_t sh) {
    return sh ? (d[i] << sh) | (d[i + 1] >> (64u - sh)) : d[i];
}

#ifndef SA_STAGED_MINB
#define SA_STAGED_MINB 4  // 4 x 256 threads per SM: 64 registers (k_match<0>'s allocation)
#endif

// part_words: words of one window's staging area (>= ceil(Lmax/32) + 3, even); slots: windows pairs
// per warp.  Dynamic shared memory: 8 warps x slots x (2 x part_words + 2) x 8 bytes.
template <int L, bool STATS>
__global__ void __launch_bounds__(256, SA_STAGED_MINB) k_match_staged(const MatchArgs a, uint32_t part_words,
                                                                    uint32_t slots) {
    extern __shared__ __align__(128) uint64_t s_stage[];
    __shared__ __align__(8) uint64_t s_bar[8];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // a slot = the read window (part_words) + the text window (part_words) + 2 pad words: the slot stride is
    // 2 mod 4 words, so the lanes' 8-byte reads at equal offsets spread over the banks (2-way at most)
    const uint32_t sw = 2 * part_words + 2;
    uint64_t *wbuf = s_stage + (uint64_t)warp * slots * sw;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar[warp]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = t < a.Q;  // (no early return: the whole warp takes part in the staged rounds)
    uint64_t q = 0, row = 0;
    uint32_t m = 0, mt = 0, lo = 0, hi = 0, steps = 0, texts = 0, ubytes = 0, ssa = 0;
    if (valid) {
        q = a.order ? (uint64_t)__ldg(a.order + t) : t;
        row = a.rows_ordered ? t : q;
        m = read_len(a, row);
        QueryWords<0> P;  // (not kept live across the staged rounds: re-loaded for a repeat's joint search)
        load_read<0>(a, row, m, P);
        ubytes = ((m + 3) >> 2) + 8;
        mt = min(m, a.k + Rec<L>::kBases);
        search_read<L, false, false>(a, P, mt, lo, hi, steps, texts, ubytes, nullptr, &ssa);  // phase (A)
    }
    const bool single = valid && m > mt && hi == lo + 1;
    uint32_t pending = __ballot_sync(0xFFFFFFFFu, single);
    uint32_t phase = 0;
    int vsign = 0;
    uint32_t vlcp = 0;
    // the read's bases as an absolute base index into the 2-bit stream a.words, and that stream's words
    const uint64_t rbase = a.stride ? 32ull * row * a.stride : (uint64_t)m * row;
    const uint64_t rtotal = a.stride ? a.Q * (uint64_t)a.stride : a.dense_words;
    const uint64_t slen = a.n - ssa;
    const uint32_t Lc = single ? (uint32_t)(min((uint64_t)m, slen) - mt) : 0u;  // bases both have past mt
    while (pending) {  // (warp-uniform)
        uint32_t sel = 0, rest = pending;
        for (uint32_t i = 0; i < slots && rest; ++i) {
            sel |= rest & (0u - rest);
            rest &= rest - 1;
        }
        pending = rest;
        const bool mine = (sel >> lane) & 1u;
        const uint32_t slot = __popc(sel & ((1u << lane) - 1u));
        uint64_t *rs = wbuf + (uint64_t)slot * sw, *ts = rs + part_words;
        StageWin gr{0, 0, 0, 0}, gt{0, 0, 0, 0};
        uint32_t bytes = 0;
        if (mine && Lc) {
            gr = stage_win(rbase + mt, Lc);
            gt = stage_win((uint64_t)ssa + mt, Lc);
            bytes = stage_bulk_bytes(gr, rtotal) + stage_bulk_bytes(gt, a.text_words);
        }
        const uint32_t total = __reduce_add_sync(0xFFFFFFFFu, bytes);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(total) : "memory");
        __syncwarp();
        if (mine && Lc) {
            // the previous round's generic-proxy reads of this slot are ordered before the async-proxy writes
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            stage_issue(rs, a.words, rtotal, gr, bar);
            stage_issue(ts, a.text, a.text_words, gt, bar);
        }
        for (uint32_t done = 0; !done;) {
            asm volatile("{ .reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2; selp.u32 %0, 1, 0, P1; }"
                         : "=r"(done) : "r"(bar), "r"(phase) : "memory");
        }
        phase ^= 1u;
        __syncwarp();  // (the plain-load tail words of every lane are visible to the warp)
#ifdef SA_STAGED_WARPCMP  // A/B: each selected lane's window pair compared by the whole warp (lane j: word j)
        for (uint32_t s2 = sel; s2;) {  // each selected lane's window pair, compared by the whole warp
            const int o = __ffs(s2) - 1;
            s2 &= s2 - 1;
            const uint32_t v = __popc(sel & ((1u << o) - 1u));
            const uint32_t oL = __shfl_sync(0xFFFFFFFFu, Lc, o);
            const uint32_t roff = __shfl_sync(0xFFFFFFFFu, gr.off, o), rsh = __shfl_sync(0xFFFFFFFFu, gr.sh, o);
            const uint32_t toff = __shfl_sync(0xFFFFFFFFu, gt.off, o), tsh = __shfl_sync(0xFFFFFFFFu, gt.sh, o);
            const uint64_t *R = wbuf + (uint64_t)v * sw, *T = R + part_words;
            const uint32_t nwL = (oL + 31) >> 5;
            int fsg = 0;
            uint32_t flc = 0xFFFFFFFFu;
            for (uint32_t j0 = 0; j0 < nwL; j0 += 32) {
                const uint32_t j = j0 + lane;
                bool dec = false;
                int sg = 0;
                uint32_t lc = 0;
                if (j < nwL) {
                    const uint64_t mask = prefix_mask(min(32u, oL - 32u * j));
                    const uint64_t x = stage_word(R, roff + j, rsh) & mask, y = stage_word(T, toff + j, tsh) & mask;
                    if (x != y) {
                        dec = true;
                        lc = 32u * j + ((uint32_t)__clzll((long long)(x ^ y)) >> 1);
                        sg = x > y ? 1 : -1;
                    }
                }
                const uint32_t b = __ballot_sync(0xFFFFFFFFu, dec);
                if (b) {
                    const int f = __ffs(b) - 1;
                    fsg = __shfl_sync(0xFFFFFFFFu, sg, f);
                    flc = __shfl_sync(0xFFFFFFFFu, lc, f);
                    break;
                }
            }
            if ((uint32_t)o == lane) {
                if (flc != 0xFFFFFFFFu) { vsign = fsg; vlcp = mt + flc; }
                else if (m <= slen) { vsign = 0; vlcp = m; }           // P is a prefix of the suffix
                else { vsign = 1; vlcp = (uint32_t)slen; }             // the suffix is a proper prefix of P (A7)
            }
        }
#else  // each selected lane compares its own window pair from shared memory, 32 bases per step
        if (mine) {
            const uint32_t nwL = (Lc + 31) >> 5;
            uint32_t j = 0;
            for (; j < nwL; ++j) {
                const uint64_t mask = prefix_mask(min(32u, Lc - 32u * j));
                const uint64_t x = stage_word(rs, gr.off + j, gr.sh) & mask, y = stage_word(ts, gt.off + j, gt.sh) & mask;
                if (x != y) {
                    vlcp = mt + 32u * j + ((uint32_t)__clzll((long long)(x ^ y)) >> 1);
                    vsign = x > y ? 1 : -1;
                    break;
                }
            }
            if (j == nwL) {
                if (m <= slen) { vsign = 0; vlcp = m; }           // P is a prefix of the suffix
                else { vsign = 1; vlcp = (uint32_t)slen; }        // the suffix is a proper prefix of P (A7)
            }
        }
#endif
        __syncwarp();
    }
    if (valid) {
        if (single) {
            ++steps;
            ++texts;
            ubytes += probe_bytes(m, mt, vlcp);
            if (vsign < 0) hi = lo;
            else if (vsign > 0) lo = hi;
        } else if (m > mt) {
            if (hi > lo) {
                QueryWords<0> P;
                load_read<0>(a, row, m, P);
                joint_search<L, false>(a, P, m, lo, hi, mt, TreeLoc{0, 0}, 0, lo, hi, steps, texts, ubytes, nullptr);
            } else {
                hi = lo;
            }
        }
        if (a.order) q = reload_u32(a.order + t);
        reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
        if (STATS) {
            a.stats[q] = min(steps, 0xFFFFu) | (min(texts, 0xFFFFu) << 16);
            a.stats[a.Q + q] = ubytes;
        }
    }
}

}  // namespace sa_search
