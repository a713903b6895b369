// encode.cu -- K4 of pipeline.compress: per-block bit lengths, block offsets, MSB-first packing
// (encode.py:117-151 symbol_bit_lengths / encode_symbols; pipeline.py:498-509).
//
//   k_enc_len   warp per block: bins staged in shared memory (coalesced 16-byte loads), lane l
//               owns the contiguous symbol range [l*c, l*c + c); per-lane bit counts, their
//               exclusive warp scan (kept for k_enc_pack) and the block total
//   k_enc_scan  decoupled look-back scan over blocks of (bits, regression records,
//               unpredictable words) -> payload bit offset, record offset, unpredictable offset
//   k_enc_pack  warp per block, 32 warps per SM: each lane packs its range at its absolute bit
//               offset into a shared-memory image of the block's big-endian 32-bit words (one
//               table load, one 64-bit shift-or per symbol, a word store every 32 bits), merged
//               with its neighbours by shared-memory ORs, then written out coalesced; words shared
//               with a neighbouring block are merged with atomicOr (k_enc_scan zeroes them)
//
// Codes come from a 4096-symbol shared window around the quantizer centre (code << 6 | len;
// code << 5 | len for the sequential packer, whose last entry is symbol 0), global memory
// outside it.  Blocks touched by bins-stage faults read their verified 32-bit
// words from fix_scratch (k_fault_bins).
namespace ftlz {

#define ENC_WIN 4096
#define SCAN_TILE 1024
#define ENC_STG 256   // payload words of a block packed through the warp's shared-memory stage

struct EncWin {
    const u64* s_enc;
    const u64* g_enc;
    int wlo, cap;
    FTLZ_DEV u64 get(u32 sym) const {
        const u32 o = sym - (u32)wlo;
        return o < (u32)ENC_WIN ? s_enc[o] : (sym < (u32)cap ? __ldg(g_enc + sym) : 0ull);
    }
    // window hit without a branch; symbols outside it (rare) take the global table
    FTLZ_DEV u64 get_fast(u32 sym) const {
        const u32 o = sym - (u32)wlo;
        u64 e = s_enc[o < (u32)ENC_WIN ? o : 0u];
        if (o >= (u32)ENC_WIN) e = sym < (u32)cap ? __ldg(g_enc + sym) : 0ull;
        return e;
    }
};

FTLZ_DEV void enc_fill_window(const CompArgs& A, u64* s_enc) {
    const int wlo = A.center - ENC_WIN / 2;
    for (int t = threadIdx.x; t < ENC_WIN; t += blockDim.x) {
        const int s = wlo + t;
        s_enc[t] = (s >= 0 && s < A.cap) ? A.enc[s] : 0ull;
    }
}

// stage block b's symbols in shared memory (u16 when read from the bins array, u32 words
// from fix_scratch for bins-faulted blocks); returns true when `sym32` holds them
FTLZ_DEV bool enc_stage(const CompArgs& A, long long b, int vol, const u32* fix, const u8* fixed_flag, u16* sym16,
                        u32* sym32, int lane) {
    const Geom& g = A.g;
    const bool fixed = A.n_faults && A.fault_first[b] >= 0 && fixed_flag[b];
    if (fixed) {
        const u32* w = fix + (size_t)b * g.vmax;
        for (int p = lane; p < vol; p += 32) sym32[p] = w[p];
    } else {
        const int nch = (vol + 7) >> 3;
        const uint4* src = (const uint4*)(A.bins + bins_index(g, b, 0));
        for (int c = lane; c < nch; c += 32) ((uint4*)sym16)[c] = __ldg(src + c);
    }
    __syncwarp();
    return fixed;
}

// next block's bins held in registers while the current block is processed (blocks of at most
// 1024 symbols, not bins-faulted): one latency per block instead of a stall before each
struct BinsPrefetch {
    uint4 r[4];
    int nch;
    FTLZ_DEV void load(const CompArgs& A, long long b, int vol, int lane) {
        nch = (vol + 7) >> 3;
        const uint4* src = (const uint4*)(A.bins + bins_index(A.g, b, 0));
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int c = lane + 32 * q;
            if (c < nch) r[q] = __ldg(src + c);
        }
    }
    FTLZ_DEV void store(u16* sym16, int lane) const {
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int c = lane + 32 * q;
            if (c < nch) ((uint4*)sym16)[c] = r[q];
        }
    }
};

FTLZ_DEV bool enc_prefetchable(const CompArgs& A, long long b, int vol, const u8* fixed_flag) {
    return vol <= 1024 && !(A.events[b] & 8) && !(A.n_faults && A.fault_first[b] >= 0 && fixed_flag[b]);
}

// code lengths of the symbols [p0, pend): a shared u8 table over the whole alphabet (no window
// test); a length of 0 marks a symbol outside the codebook (pipeline.py:490)
FTLZ_DEV u32 len_range(const u8* s_len, const u16* sym16, int p0, int pend, bool& range_err) {
    u32 bits = 0, zero = 0;
#pragma unroll 4
    for (int p = p0; p < pend; p++) {
        const u32 l = s_len[sym16[p]];
        zero |= (u32)(l == 0u);
        bits += l;
    }
    range_err |= zero != 0;
    return bits;
}
// bins-faulted blocks: 32-bit words straight from fix_scratch (rare path)
FTLZ_DEV u32 len_range_fixed(const u8* s_len, int cap, const u32* w, int p0, int pend, bool& range_err) {
    u32 bits = 0;
    for (int p = p0; p < pend; p++) {
        const u32 sym = w[p];
        const u32 l = sym < (u32)cap ? s_len[sym] : 0u;
        range_err |= l == 0u;
        bits += l ? l : 1u;
    }
    return bits;
}

__global__ void __launch_bounds__(512) k_enc_len(CompArgs A, const u32* fix, const u8* fixed_flag, const u8* lens) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (dev_failed(A.st)) return;
    const Geom& g = A.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int capal = (A.cap + 15) & ~15;
    u8* s_len = smem;
    u16* sym16 = (u16*)(smem + capal + (size_t)warp * 2 * g.nvmax8);
    for (int t = threadIdx.x; t < capal / 16; t += blockDim.x)
        ((uint4*)s_len)[t] = t * 16 + 16 <= A.cap ? __ldg((const uint4*)lens + t) : make_uint4(0, 0, 0, 0);
    for (int t = (A.cap & ~15) + threadIdx.x; t < A.cap; t += blockDim.x) s_len[t] = lens[t];
    __syncthreads();
    const long long NW = (long long)gridDim.x * nw;
    long long b = (long long)blockIdx.x * nw + warp;
    BinsPrefetch P;
    bool pf = false;
    int vol = 0;
    if (b < g.nb) {
        vol = block_info(g, b).vol;
        pf = enc_prefetchable(A, b, vol, fixed_flag);
        if (pf) P.load(A, b, vol, lane);
    }
    for (; b < g.nb; b += NW) {
        u32 bits = 0;
        bool range_err = false;
        const bool bad = (A.events[b] & 8) != 0;
        const bool fixed = !bad && A.n_faults && A.fault_first[b] >= 0 && fixed_flag[b];
        if (!bad && !fixed) {
            if (pf) P.store(sym16, lane);
            else {
                const int nch = (vol + 7) >> 3;
                const uint4* src = (const uint4*)(A.bins + bins_index(g, b, 0));
                for (int c = lane; c < nch; c += 32) ((uint4*)sym16)[c] = __ldg(src + c);
            }
        }
        __syncwarp();
        const int cvol = vol;
        const long long bn = b + NW;
        if (bn < g.nb) {
            vol = block_info(g, bn).vol;
            pf = enc_prefetchable(A, bn, vol, fixed_flag);
            if (pf) P.load(A, bn, vol, lane);
        }
        if (!bad) {
            const int chunk = ((cvol + 31) >> 5) | 1;
            const int p0 = lane * chunk, pend = min(p0 + chunk, cvol);
            if (fixed) bits = len_range_fixed(s_len, A.cap, fix + (size_t)b * g.vmax, p0, pend, range_err);
            else bits = len_range(s_len, sym16, p0, pend, range_err);
        }
        __syncwarp();
        u32 pre = bits;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += v;
        }
        A.lanepre[(size_t)b * 32 + lane] = pre - bits;
        if (lane == 31) A.bitlen[b] = pre;
        if (__any_sync(0xffffffffu, range_err) && lane == 0)
            dev_fail(A.st, FTLZ_ERR_INVARIANT, FTLZ_K_BIN_RANGE, -1, b, 0, 0, 0);
    }
}

// exclusive scans over blocks: payload bits (u64), regression records, unpredictable words
__global__ void __launch_bounds__(SCAN_TILE) k_enc_scan(CompArgs A, u32* lb_flag, u64* lb_bits, u64* lb_reg, u64* lb_unp) {
    if (dev_failed(A.st)) return;
    const Geom& g = A.g;
    __shared__ u64 s_w[3][SCAN_TILE / 32];
    __shared__ u64 s_pre[3];
    __shared__ unsigned s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    if (tid == 0) s_tile = atomicAdd(&A.counters[2], 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const long long b = (long long)tile * SCAN_TILE + tid;
    const bool valid = b < g.nb;
    u64 v3[3] = {valid ? (u64)A.bitlen[b] : 0ull, valid ? (u64)A.ind[b] : 0ull, valid ? (u64)A.unpc[b] : 0ull};
    u64 inc[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        inc[q] = v3[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u64 t = __shfl_up_sync(0xffffffffu, inc[q], o);
            if (lane >= o) inc[q] += t;
        }
        if (lane == 31) s_w[q][warp] = inc[q];
    }
    __syncthreads();
    u64 woff[3] = {0, 0, 0}, tsum[3] = {0, 0, 0};
#pragma unroll
    for (int q = 0; q < 3; q++)
        for (int w = 0; w < nwarp; w++) {
            if (w < warp) woff[q] += s_w[q][w];
            tsum[q] += s_w[q][w];
        }
    if (warp == 0) {
        // flag: 0 = empty, 1 = aggregate published, 2 = inclusive prefix published.  Look-back
        // by the whole warp: lane l reads tile (t - l); the nearest inclusive prefix ends it.
        volatile u64* vb = lb_bits;
        volatile u64* vr = lb_reg;
        volatile u64* vu = lb_unp;
        volatile u32* vf = lb_flag;
        u64 pre[3] = {0, 0, 0};
        if (tile > 0) {
            if (lane == 0) {
                vb[2 * tile] = tsum[0];
                vr[2 * tile] = tsum[1];
                vu[2 * tile] = tsum[2];
                __threadfence();
                vf[tile] = 1;
            }
            long long t = (long long)tile - 1;
            while (t >= 0) {
                const long long ti = t - lane;
                const u32 f = ti >= 0 ? vf[ti] : 3u;   // 3: before tile 0 (an empty inclusive prefix)
                const unsigned incl = __ballot_sync(0xffffffffu, f >= 2u);
                const unsigned zero = __ballot_sync(0xffffffffu, f == 0u);
                const int fi = incl ? __ffs(incl) - 1 : 32;
                const unsigned need = fi == 32 ? 0xffffffffu : ((2u << fi) - 1u);
                if (zero & need) continue;
                __threadfence();
                u64 a[3] = {0, 0, 0};
                const int sl = lane < fi ? 0 : 1;
                if (lane < fi || (lane == fi && f == 2u)) {
                    a[0] = vb[2 * ti + sl];
                    a[1] = vr[2 * ti + sl];
                    a[2] = vu[2 * ti + sl];
                }
#pragma unroll
                for (int q = 0; q < 3; q++) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
                    pre[q] += a[q];
                }
                if (fi < 32) break;
                t -= 32;
            }
        }
        if (lane == 0) {
            vb[2 * tile + 1] = pre[0] + tsum[0];
            vr[2 * tile + 1] = pre[1] + tsum[1];
            vu[2 * tile + 1] = pre[2] + tsum[2];
            __threadfence();
            vf[tile] = 2;
            s_pre[0] = pre[0];
            s_pre[1] = pre[1];
            s_pre[2] = pre[2];
        }
    }
    __syncthreads();
    if (!valid) return;
    const u64 boff = s_pre[0] + woff[0] + inc[0] - v3[0];
    // zero the payload words k_enc_pack merges with atomicOr (k_enc_pack runs after this
    // kernel): the first and last word of every block (shared with its neighbours)
    {
        u32* words = (u32*)A.out;
        const u64 bpos = A.layout[LAYOUT_PAY_OFF] * 8 + boff;
        const u64 w0 = bpos >> 5, w1 = (bpos + v3[0] + 31) >> 5;
        if (w1 > w0) {   // (the interior of an unstaged block is zeroed by its own warp in k_enc_pack)
            words[w0] = 0u;
            words[w1 - 1] = 0u;
        }
    }
    A.bitoff[b] = boff;
    A.regpre[b] = (u32)(s_pre[1] + woff[1] + inc[1] - v3[1]);
    A.unppre[b] = s_pre[2] + woff[2] + inc[2] - v3[2];
}

// one big-endian word of the payload (u32 index into the archive): atomicOr when shared
FTLZ_DEV void enc_put(u32* words, u64 widx, u32 bits_be, bool shared_word) {
    const u32 v = __byte_perm(bits_be, 0, 0x0123);
    if (shared_word) atomicOr(words + widx, v);
    else words[widx] = v;
}

// predicated form for the packing loop (no divergent branch): p_st plain store, p_or atomic OR
FTLZ_DEV void enc_put_pred(u32* addr, u32 bits_be, bool p_st, bool p_or) {
    const u32 v = __byte_perm(bits_be, 0, 0x0123);
    asm volatile(
        "{\n\t.reg .pred a, b;\n\tsetp.ne.u32 a, %2, 0;\n\tsetp.ne.u32 b, %3, 0;\n\t"
        "@a st.global.u32 [%0], %1;\n\t@b red.global.or.b32 [%0], %1;\n\t}"
        ::"l"(addr), "r"(v), "r"((u32)p_st), "r"((u32)p_or)
        : "memory");
}

// MSB-first packing of symbols [p0, pend) starting at absolute bit gpos; FIXED: 32-bit symbols
// of a bins-faulted block; LONG: some code is longer than 32 bits
template <bool FIXED, bool LONG>
FTLZ_DEV void pack_range(const EncWin& W, const u16* sym16, const u32* sym32, int p0, int pend, u64 gpos, u32* words) {
    u64 widx = gpos >> 5;
    u64 acc = 0;                          // pending bits, left-aligned at bit 63
    int nacc = (int)(gpos & 31);          // leading bits of the first word belong to others
    bool first = true;
    for (int p = p0; p < pend; p++) {
        const u32 sym = FIXED ? sym32[p] : (u32)sym16[p];
        const u64 e = W.get_fast(sym);
        int l = (int)(e & 63);
        u64 code = e >> 6;
        if (LONG && l > 32) {
            const int hl = l - 32;
            acc |= (code >> 32) << (64 - nacc - hl);
            nacc += hl;
            if (nacc >= 32) {
                enc_put(words, widx++, (u32)(acc >> 32), first);
                first = false;
                acc <<= 32;
                nacc -= 32;
            }
            code &= 0xffffffffull;
            l = 32;
        }
        acc |= code << (64 - nacc - l);
        nacc += l;
        // full word: store it (atomic OR for the lane's first word, shared with the lane or
        // block before), predicated instead of branched
        const bool full = nacc >= 32;
        enc_put_pred(words + widx, (u32)(acc >> 32), full && !first, full && first);
        first = first && !full;
        widx += full ? 1 : 0;
        acc = full ? acc << 32 : acc;
        nacc -= full ? 32 : 0;
    }
    if (nacc > 0) enc_put(words, widx, (u32)(acc >> 32), true);
}

// the same packing into a warp's shared staging buffer (word 0 = the block's first payload
// word); words shared between lanes are merged with shared-memory ORs
FTLZ_DEV void put_s(u32 addr, u32 bits_be, bool p_st, bool p_or) {
    const u32 v = __byte_perm(bits_be, 0, 0x0123);
    asm volatile(
        "{\n\t.reg .pred a, b;\n\tsetp.ne.u32 a, %2, 0;\n\tsetp.ne.u32 b, %3, 0;\n\t"
        "@a st.shared.u32 [%0], %1;\n\t@b red.shared.or.b32 [%0], %1;\n\t}"
        ::"r"(addr), "r"(v), "r"((u32)p_st), "r"((u32)p_or)
        : "memory");
}

template <bool FIXED, bool LONG>
FTLZ_DEV void pack_range_s(const EncWin& W, const u16* sym16, const u32* sym32, int p0, int pend, u32 pos, u32 sbase) {
    u32 widx = pos >> 5;
    u64 acc = 0;
    int nacc = (int)(pos & 31);
    bool first = true;
    for (int p = p0; p < pend; p++) {
        const u32 sym = FIXED ? sym32[p] : (u32)sym16[p];
        const u64 e = W.get_fast(sym);
        int l = (int)(e & 63);
        u64 code = e >> 6;
        if (LONG && l > 32) {
            const int hl = l - 32;
            acc |= (code >> 32) << (64 - nacc - hl);
            nacc += hl;
            const bool f1 = nacc >= 32;
            put_s(sbase + 4u * widx, (u32)(acc >> 32), f1 && !first, f1 && first);
            first = first && !f1;
            widx += f1 ? 1u : 0u;
            acc = f1 ? acc << 32 : acc;
            nacc -= f1 ? 32 : 0;
            code &= 0xffffffffull;
            l = 32;
        }
        acc |= code << (64 - nacc - l);
        nacc += l;
        const bool full = nacc >= 32;
        put_s(sbase + 4u * widx, (u32)(acc >> 32), full && !first, full && first);
        first = first && !full;
        widx += full ? 1u : 0u;
        acc = full ? acc << 32 : acc;
        nacc -= full ? 32 : 0;
    }
    if (nacc > 0) put_s(sbase + 4u * widx, (u32)(acc >> 32), false, true);
}

#define C32_BYTES ((4 * (ENC_WIN + 1) + 15) & ~15)   // k_enc_pack's code << 5 | len window

// sequential MSB-first packing of symbols [p0, pend) into the warp's staged words, for
// alphabets whose nonzero symbols all lie in the window (code << 5 | len entries, codes of at
// most 27 bits; entry ENC_WIN is symbol 0, every other symbol maps into the window): per
// symbol one table load, a 64-bit shift-or and, every 32 bits, one predicated word store
// (the lane's first word, shared with the lane before, is merged with a shared-memory OR)
FTLZ_DEV void pack_range_seq(const u32* s_c32, int wlo, const u16* sym16, int p0, int pend, u32 pos, u32 sbase) {
    u32 waddr = sbase + 4u * (pos >> 5);   // shared address of the word being filled
    u32 nacc = pos & 31;   // bits of the first word that belong to the lanes before (zero in acc)
    u64 acc = 0;           // pending bits, right-aligned
    int p = p0;
    // up to the lane's first full word (shared with the lane before: shared-memory OR)
    for (; p < pend; p++) {
        const u32 e = s_c32[min((u32)sym16[p] - (u32)wlo, (u32)ENC_WIN)];
        const u32 l = e & 31u;
        acc = (acc << l) | (u64)(e >> 5);
        nacc += l;
        if (nacc >= 32u) {
            nacc -= 32u;
            put_s(waddr, (u32)(acc >> nacc), false, true);
            waddr += 4u;
            p++;
            break;
        }
    }
    // the lane's own words: plain predicated stores
#pragma unroll 2
    for (; p < pend; p++) {
        const u32 e = s_c32[min((u32)sym16[p] - (u32)wlo, (u32)ENC_WIN)];
        const u32 l = e & 31u;
        acc = (acc << l) | (u64)(e >> 5);
        nacc += l;
        const bool full = nacc >= 32u;
        nacc -= full ? 32u : 0u;
        const u32 v = __byte_perm((u32)(acc >> nacc), 0, 0x0123);
        asm volatile("{\n\t.reg .pred a;\n\tsetp.ne.u32 a, %2, 0;\n\t@a st.shared.u32 [%0], %1;\n\t}"
                     ::"r"(waddr), "r"(v), "r"((u32)full) : "memory");
        waddr += full ? 4u : 0u;
    }
    if (nacc > 0u) put_s(waddr, (u32)(acc << (32u - nacc)), false, true);
}

__global__ void __launch_bounds__(1024) k_enc_pack(CompArgs A, const u32* fix, const u8* fixed_flag) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (dev_failed(A.st)) return;
    const Geom& g = A.g;
    u64* s_enc = (u64*)smem;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    u32* s_c32 = (u32*)(smem + 8 * ENC_WIN);   // ENC_WIN + 1 entries (code << 5 | len; last: symbol 0)
    u16* sym16 = (u16*)(smem + 8 * ENC_WIN + C32_BYTES + (size_t)warp * 2 * g.nvmax8);
    u32* stg = (u32*)(smem + 8 * ENC_WIN + C32_BYTES + (size_t)nw * 2 * g.nvmax8) + (size_t)warp * ENC_STG;
    const u32 stg_sa = smem_u32(stg);
    const int wlo = A.center - ENC_WIN / 2;
    enc_fill_window(A, s_enc);
    for (int t = threadIdx.x; t <= ENC_WIN; t += blockDim.x) {
        const int sy = t == ENC_WIN ? 0 : wlo + t;
        const u64 e = (sy >= 0 && sy < A.cap) ? A.enc[sy] : 0ull;
        s_c32[t] = (u32)((e >> 6) << 5) | (u32)(e & 31);
    }
    // every nonzero symbol inside the window and codes of at most 26 bits: sequential packer
    const bool seq = A.layout[LAYOUT_MAXLEN] <= 27 && A.layout[LAYOUT_SYMLO] >= (u64)(wlo > 0 ? wlo : 0) &&
                     A.layout[LAYOUT_SYMHI] < (u64)(wlo + ENC_WIN) && wlo > 0;
    __syncthreads();
    const EncWin W = {s_enc, A.enc, A.center - ENC_WIN / 2, A.cap};
    u32* words = (u32*)A.out;
    const u64 pay0 = A.layout[LAYOUT_PAY_OFF] * 8;
    const bool longc = A.layout[LAYOUT_MAXLEN] > 32;
    const long long NW = (long long)gridDim.x * nw;
    long long b = (long long)blockIdx.x * nw + warp;
    BinsPrefetch P;
    bool pf = false;
    int nvol = 0;
    if (b < g.nb) {
        nvol = block_info(g, b).vol;
        pf = enc_prefetchable(A, b, nvol, fixed_flag);
        if (pf) P.load(A, b, nvol, lane);
    }
    for (; b < g.nb; b += NW) {
        const int vol = nvol;
        const bool bad = (A.events[b] & 8) != 0;
        const bool fixed = !bad && A.n_faults && A.fault_first[b] >= 0 && fixed_flag[b];
        // bins-faulted blocks pack their verified 32-bit words straight from fix_scratch
        const u32* sym32 = fix + (size_t)b * g.vmax;
        if (!bad && !fixed) {
            if (pf) P.store(sym16, lane);
            else {
                const int nch = (vol + 7) >> 3;
                const uint4* src = (const uint4*)(A.bins + bins_index(g, b, 0));
                for (int c = lane; c < nch; c += 32) ((uint4*)sym16)[c] = __ldg(src + c);
            }
        }
        __syncwarp();
        const long long bn = b + NW;
        if (bn < g.nb) {
            nvol = block_info(g, bn).vol;
            pf = enc_prefetchable(A, bn, nvol, fixed_flag);
            if (pf) P.load(A, bn, nvol, lane);
        }
        if (bad) continue;
        const int chunk = ((vol + 31) >> 5) | 1;
        const int p0 = lane * chunk, pend = min(p0 + chunk, vol);
        const u64 bpos = pay0 + A.bitoff[b];
        const u64 gpos = bpos + A.lanepre[(size_t)b * 32 + lane];
        const u64 w0 = bpos >> 5, nwords = ((bpos + A.bitlen[b] + 31) >> 5) - w0;
        if (nwords <= ENC_STG) {
            // staged: the block's words assembled in shared memory, then written coalesced
            // (its first and last words are shared with the neighbouring blocks: atomic OR)
            for (int i = lane; i < (int)nwords; i += 32) stg[i] = 0;
            __syncwarp();
            const u32 pos = (u32)(gpos - w0 * 32);
            if (p0 < pend) {
                if (fixed) pack_range_s<true, true>(W, sym16, sym32, p0, pend, pos, stg_sa);
                else if (seq) pack_range_seq(s_c32, wlo, sym16, p0, pend, pos, stg_sa);
                else if (longc) pack_range_s<false, true>(W, sym16, sym32, p0, pend, pos, stg_sa);
                else pack_range_s<false, false>(W, sym16, sym32, p0, pend, pos, stg_sa);
            }
            __syncwarp();
            for (int i = lane; i < (int)nwords; i += 32) {
                const u32 v = stg[i];
                if (i == 0 || i == (int)nwords - 1) atomicOr(words + w0 + i, v);
                else words[w0 + i] = v;
            }
        } else {
            // unstaged: this warp zeroes the block's interior words (lanes merge at their range
            // boundaries), coalesced, before packing in place
            for (u64 i = w0 + 1 + lane; i + 1 < w0 + nwords; i += 32) words[i] = 0u;
            __threadfence();   // the zeros reach L2 before any lane's atomicOr on them
            __syncwarp();
        }
        if (nwords > ENC_STG && p0 < pend) {
            if (fixed) pack_range<true, true>(W, sym16, sym32, p0, pend, gpos, words);
            else if (longc) pack_range<false, true>(W, sym16, sym32, p0, pend, gpos, words);
            else pack_range<false, false>(W, sym16, sym32, p0, pend, gpos, words);
        }
        __syncwarp();
    }
}

}  // namespace ftlz
