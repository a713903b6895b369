// decode_warp.cu -- the fault-free full decode with a warp per block: _Decoder
// (encode.py:168-256) + _reconstruct_group of regression blocks (pipeline.py:586-638) + the
// sum_dc verification (pipeline.py:692-707) for the default block edge (10).
//
// k_decode gives each lane a whole block, so a block's 1000 codes are one serial chain: small
// fields run out of blocks long before they run out of lanes, and on large ones every refill of a
// lane's bit window waits on the latest global load of any lane of its warp.  Here the 32 lanes
// of a warp split ONE block's bit slice, staged in shared memory, with self-synchronising
// (speculative) Huffman decoding:
//   1. lane l decodes from bit l * seg of the slice (seg a multiple of 32), marking every code
//      boundary it meets inside its segment in a bitmap, up to its exit: the first boundary at or
//      past the segment end.  Lane 0 starts on a true boundary, so its path is the true one.
//   2. the true path enters segment l at the exit of lane l - 1.  From there lane l decodes until
//      it lands on one of its own marked boundaries: both paths coincide from that point, so its
//      true symbol count is what it decoded plus the marked boundaries left in its segment, and
//      its exit is the speculative one.  A lane that never lands on a mark (rare) decodes to its
//      segment end and hands its new exit on; the pass repeats until no entry point moves.
//   3. with every lane's entry point and symbol count known (prefix sum: output index), each
//      lane decodes its symbols again into a shared-memory symbol array, two per look-up of a
//      12-bit table when both codes fit.
//   4. the warp reconstructs the block from the symbol array, 32 consecutive points at a time
//      (regression blocks; Lorenzo blocks copy their bins to scratch for k_recon_g), counts the
//      unpredictable points by ballot, and verifies sum_dc.
// The slice words are byte-swapped once while staged, so every window is a funnel shift of
// shared words.  A block whose decode is anything but clean (a code outside the code space, a
// wrong symbol count, a slice not consumed exactly, a wrong unpredictable count) is marked
// DF_PENDING for the masked reader to classify, as k_decode's fast path does.  A block whose
// slice exceeds the staging buffer (more than ~16 bits per point) is decoded by lane 0 alone from
// global memory.
namespace ftlz {

#define PAIR_TBITS 12
#define DW_WARPS 24
#define DW_SW 448           // staged slice words per warp (14 bits per point)
#define DW_E 10
#define DW_VMAX 1024        // symbol slots (>= 10^3)
#define DW_LONGSYM 1024     // symbols of codes longer than the table kept in shared memory

// decode LUTs: T-bit window -> (symbol << 8 | length) for codes of length <= T (0: longer); the
// window's length is the first l with x < end_l = (F_l + count_l) << (T - l), which is
// non-decreasing in l (binary search).  Grid-wide, one launch: the 2^T-entry table of the
// full-path decoder, the 2^T12-entry table of the list decodes and, for the warp-per-block
// decoder (pairs != 0), its 2^PAIR_TBITS-entry pair table.
//
// pair table entry: bits 0-5 bits consumed, 6-7 symbol count n (0: first code longer than the
// table or outside the code space), 8-13 length of the first code, 16-31 first symbol, 32-47
// second symbol, 48-59 start offsets of the codes lying wholly inside the window, 60-63 the bits
// they cover (0: first code longer than the table)
__global__ void __launch_bounds__(256) k_dec_luts(DecArgs A, int pairs) {
    if (dev_failed(A.st)) return;
    __shared__ u64 s_fc[64];
    __shared__ u32 s_lc[64], s_lb[64];
    if (threadIdx.x < 64) { s_fc[threadIdx.x] = A.first_code[threadIdx.x]; s_lc[threadIdx.x] = A.lcount[threadIdx.x]; s_lb[threadIdx.x] = A.lbase[threadIdx.x]; }
    __syncthreads();
    const int T = (int)A.info[DI_T], T12 = (int)A.info[DI_T12];
    const u32 n1 = 1u << T, n2 = 1u << T12, n3 = pairs ? 1u << PAIR_TBITS : 0u;
    // the code at the head of the TT-bit window x: symbol << 8 | length, 0 if longer than TT
    auto look = [&](u32 x, int TT) -> u32 {
        int lo = 1, hi = TT + 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((u64)x < ((s_fc[mid] + s_lc[mid]) << (TT - mid))) hi = mid;
            else lo = mid + 1;
        }
        return lo <= TT ? (A.dsym[s_lb[lo] + (u32)((u64)(x >> (TT - lo)) - s_fc[lo])] << 8) | (u32)lo : 0u;
    };
    for (u32 t = blockIdx.x * blockDim.x + threadIdx.x; t < n1 + n2 + n3; t += gridDim.x * blockDim.x) {
        if (t < n1) { A.lut[t] = look(t, T); continue; }
        if (t < n1 + n2) { A.lut12[t - n1] = look(t - n1, T12); continue; }
        const u32 v = t - n1 - n2, M = (1u << PAIR_TBITS) - 1u;
        // a code wholly inside the top `nvalid` bits of the PAIR_TBITS-bit window u
        auto pl = [&](u32 u, int nvalid) -> u32 {
            const u32 e = look(u, PAIR_TBITS);
            return (e && (int)(e & 63u) <= nvalid) ? e : 0u;
        };
        const u32 e1 = pl(v, PAIR_TBITS);
        u64 ent = 0;
        if (e1) {
            const u32 l1 = e1 & 63u, s1 = e1 >> 8;
            const u32 e2 = pl((v << l1) & M, PAIR_TBITS - (int)l1);
            if (e2) {
                const u32 l2 = e2 & 63u, s2 = e2 >> 8;
                ent = (u64)(l1 + l2) | (2ull << 6) | ((u64)l1 << 8) | ((u64)s1 << 16) | ((u64)s2 << 32);
            } else {
                ent = (u64)l1 | (1ull << 6) | ((u64)l1 << 8) | ((u64)s1 << 16);
            }
            u32 off = 0, mask = 0;
            while (off < PAIR_TBITS) {
                const u32 e = pl((v << off) & M, PAIR_TBITS - (int)off);
                if (!e) break;
                mask |= 1u << off;
                off += e & 63u;
            }
            ent |= ((u64)mask << 48) | ((u64)off << 60);
        }
        A.lut2[v] = ent;
    }
}

FTLZ_DEV u64 lds_u64(u32 addr) {
    u64 v;
    asm("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}

// canonical tables of the long-code path (codes longer than the pair table)
__shared__ u64 s_dw_first[64];
__shared__ u32 s_dw_count[64], s_dw_base[64];
__shared__ u32 s_dw_lsym[DW_LONGSYM];
__shared__ u32 s_dw_lbase, s_dw_lall;
__shared__ int s_dw_maxlen;

__device__ __noinline__ u32 dw_dsym_global(const u32* dsym, u32 idx) { return dsym[idx]; }

// a code longer than the table at the head of the 64-bit window w: its length (0: outside the
// code space) and symbol
FTLZ_DEV int dw_long(u64 w, const u32* dsym, u32& sym) {
    for (int l = PAIR_TBITS + 1; l <= s_dw_maxlen; l++) {
        const u64 d = (w >> (64 - l)) - s_dw_first[l];
        if (d < (u64)s_dw_count[l]) {
            const u32 idx = s_dw_base[l] + (u32)d;
            sym = s_dw_lall ? s_dw_lsym[idx - s_dw_lbase] : dw_dsym_global(dsym, idx);
            return l;
        }
    }
    return 0;
}

// windows over the staged (byte-swapped) slice words at bit x
FTLZ_DEV u32 dw_win32(const u32* sb, u32 x) { return __funnelshift_l(sb[(x >> 5) + 1], sb[x >> 5], x & 31); }
FTLZ_DEV u64 dw_win64(const u32* sb, u32 x) {
    const u32 n = x >> 5, s = x & 31;
    const u32 a = sb[n], b = sb[n + 1], c = sb[n + 2];
    return ((u64)__funnelshift_l(b, a, s) << 32) | __funnelshift_l(c, b, s);
}

// length of the code at bit x (0: outside the code space)
FTLZ_DEV int dw_len(const u32* sb, u32 x, u32 tab_sa, const u32* dsym) {
    const u64 ent = lds_u64(tab_sa + 8u * (dw_win32(sb, x) >> (32 - PAIR_TBITS)));
    if ((u32)ent & 0xc0u) return (int)(ent >> 8) & 63;
    u32 sym;
    return dw_long(dw_win64(sb, x), dsym, sym);
}

// one symbol at bit x: its length (0: outside the code space)
FTLZ_DEV int dw_sym(const u32* sb, u32 x, u32 tab_sa, const u32* dsym, u32& sym) {
    const u64 ent = lds_u64(tab_sa + 8u * (dw_win32(sb, x) >> (32 - PAIR_TBITS)));
    if ((u32)ent & 0xc0u) {
        sym = (u32)(ent >> 16) & 0xffffu;
        return (int)(ent >> 8) & 63;
    }
    return dw_long(dw_win64(sb, x), dsym, sym);
}

// marked boundaries of the bitmap in [p, e) (p < e)
FTLZ_DEV u32 dw_popc_range(const u32* bm, u32 p, u32 e) {
    u32 c = 0;
    const u32 w1 = (e - 1) >> 5;
    for (u32 wi = p >> 5; wi <= w1; wi++) {
        u32 v = bm[wi];
        if (wi == (p >> 5)) v &= ~0u << (p & 31);
        if (wi == w1 && (e & 31)) v &= (1u << (e & 31)) - 1u;
        c += __popc(v);
    }
    return c;
}

struct DwSlot {
    u32 sb[DW_SW + 4];
    u32 bm[DW_SW];
    union {
        u16 sym[DW_VMAX];   // pass 3, reconstruction
        u32 tm[DW_SW];      // synchronisation: boundaries of the true path
    };
    union {
        double ab[DW_E * DW_E];   // reconstruction
        u16 wpre[DW_SW];          // symbols before each bitmap word
    };
    double ck[16];
    long long rowoff[DW_E * DW_E];   // output offset of each row of the block
};
#define DW_SMEM (((size_t)8 << PAIR_TBITS) + (size_t)DW_WARPS * sizeof(DwSlot))

__global__ void __launch_bounds__(DW_WARPS * 32, 1) k_decode_warp(DecArgs A) {
    if (dev_failed(A.st)) return;
    extern __shared__ __align__(16) u64 ptab[];
    const Geom& g = A.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {
        const uint4* src = (const uint4*)A.lut2;
        uint4* dst = (uint4*)ptab;
        for (int x = tid; x < (1 << PAIR_TBITS) / 2; x += blockDim.x) dst[x] = src[x];
    }
    const int maxlen = (int)A.info[DI_MAXLEN], nsym = (int)A.info[DI_NSYM];
    if (tid < 64) { s_dw_first[tid] = A.first_code[tid]; s_dw_count[tid] = A.lcount[tid]; s_dw_base[tid] = A.lbase[tid]; }
    {
        const u32 lb = maxlen > PAIR_TBITS ? A.lbase[PAIR_TBITS + 1] : (u32)nsym;
        if (tid == 0) { s_dw_lbase = lb; s_dw_lall = (u32)nsym - lb <= DW_LONGSYM; s_dw_maxlen = maxlen; }
        for (int x = tid; x < DW_LONGSYM && lb + (u32)x < (u32)nsym; x += blockDim.x) s_dw_lsym[x] = A.dsym[lb + x];
    }
    __syncthreads();
    u32 tab_sa;
    asm volatile("mov.u32 %0, %1;" : "=r"(tab_sa) : "r"(smem_u32(ptab)));
    DwSlot& S = *(DwSlot*)((unsigned char*)ptab + ((size_t)8 << PAIR_TBITS) + (size_t)warp * sizeof(DwSlot));
    const u64 pay_off = pay_boff(A), pay_len = A.info[DI_PAY_LEN];
    const u64 bufw = ((A.codec ? A.pay_cap : A.len) + 3) >> 2;
    const u32* pay_words = (const u32*)pay_base(A);
    const double twoeb = A.twoeb;
    const int center = A.center;
    const long long plane = g.ny * g.nz;
    const bool has_sdc = A.info[DI_HAS_SDC] != 0;
    const unsigned FULL = 0xffffffffu;
    const u32 nblk = (u32)(A.sb1 - A.sb0);

    for (;;) {
        u32 t = 0;
        if (lane == 0) t = atomicAdd(&A.counters[DC_DTICKET], 1u);
        t = __shfl_sync(FULL, t, 0);
        if (t >= nblk) break;
        const long long b = A.sb0 + t;
        const BlockInfo B = block_info(g, b);
        const int bz = B.bz, by = B.by, vol = B.vol, nrows = B.bx * B.by;
        const bool recon = A.ind[b] == 1;
        const u32 bl = A.bitlen[b];
        const u64 rel = A.bofs[b];
        if (((rel + bl + 7) >> 3) > pay_len) {
            if (lane == 0) fail_block(A, b, FTLZ_K_D_PAST_END, 0, 0);
            continue;
        }
        const u64 start = pay_off * 8 + rel;
        const u64 w0 = start >> 5;
        const u32 P0 = (u32)(start & 31);
        const u32 nwords = (P0 + bl + 31) >> 5;
        bool bad = false;   // warp-uniform after the decode
        if (nwords + 3 <= DW_SW) {
            // ---- stage the slice (byte-swapped; three zero-padded guard words), clear the bitmap
            for (u32 x = lane; x < nwords + 3; x += 32) {
                const u64 wi = w0 + x;
                S.sb[x] = wi < bufw ? __byte_perm(__ldg(pay_words + wi), 0, 0x0123) : 0u;
            }
            const u32 seg = ((bl + 1023) >> 10) << 5;   // bits per lane, a multiple of 32
            const u32 sw = seg >> 5;                   // bitmap words per lane
            for (u32 x = lane; x < seg; x += 32) S.bm[x] = 0;   // 32 lanes x sw words
            __syncwarp();
            // ---- 1. speculative pass, several codes per look-up (work follows bits, not codes)
            const u32 q0 = lane * seg, qend = min(q0 + seg, bl);
            u32 E = q0, cnt = 0;
            bool sok = true;
            if (q0 < bl) {
                u32 q = q0, cw = q0 >> 5;
                u64 acc = 0;
                while (q < qend) {
                    u32 sh = q - cw * 32;
                    while (sh >= 32) {
                        S.bm[cw] = (u32)acc;
                        acc >>= 32;
                        cw++;
                        sh -= 32;
                    }
                    const u32 x = P0 + q;
                    const u64 ent = lds_u64(tab_sa + 8u * (dw_win32(S.sb, x) >> (32 - PAIR_TBITS)));
                    const u32 tot = (u32)(ent >> 60);
                    if (tot == 0) {
                        u32 sym;
                        const int l = dw_long(dw_win64(S.sb, x), A.dsym, sym);
                        if (!l) { sok = false; break; }
                        acc |= 1ull << sh;
                        q += (u32)l;
                        cnt++;
                        continue;
                    }
                    const u32 mask = (u32)(ent >> 48) & 0xfffu, room = qend - q;
                    if (room < tot) {
                        // last look-up: marks below qend; exit at the first boundary at or past it
                        const u32 keep = mask & ((1u << room) - 1u), rest = mask >> room;
                        acc |= (u64)keep << sh;
                        cnt += __popc(keep);
                        q = rest ? q + room + (u32)(__ffs(rest) - 1) : q + tot;
                        break;
                    }
                    acc |= (u64)mask << sh;
                    cnt += __popc(mask);
                    q += tot;
                }
                // own words are [q0 / 32, q0 / 32 + sw); marks lie below qend
                S.bm[cw] = (u32)acc;
                if (cw + 1 < (q0 >> 5) + sw) S.bm[cw + 1] = (u32)(acc >> 32);
                E = q;
            }
            __syncwarp();
            // ---- 2. synchronisation; the true path's boundaries before the meeting point go to tm
            u32 tin = __shfl_up_sync(FULL, E, 1);
            if (lane == 0) tin = 0;
            const bool walker = q0 < bl && lane > 0;
            u32 c = cnt, Eout = E, meet = q0;
            bool lbad = !sok, synced = true;
            for (int it = 0; it < 33; it++) {
                if (q0 >= bl) { c = 0; Eout = tin; lbad = false; }
                else if (walker) {
                    for (u32 x = 0; x < sw; x++) S.tm[(q0 >> 5) + x] = 0;
                    lbad = false;
                    synced = false;
                    u32 pos = tin, a = 0;
                    while (pos < qend) {
                        if ((S.bm[pos >> 5] >> (pos & 31)) & 1u) { synced = true; break; }
                        S.tm[pos >> 5] |= 1u << (pos & 31);
                        const int l = dw_len(S.sb, P0 + pos, tab_sa, A.dsym);
                        if (!l) { lbad = true; break; }
                        pos += (u32)l;
                        a++;
                    }
                    meet = pos;
                    if (synced) {
                        c = a + dw_popc_range(S.bm, pos, qend);
                        Eout = E;
                        lbad = lbad || !sok;
                    } else {
                        c = a;
                        Eout = pos;
                    }
                }
                u32 nt = __shfl_up_sync(FULL, Eout, 1);
                if (lane == 0) nt = 0;
                if (__all_sync(FULL, !walker || nt == tin)) break;
                tin = nt;
            }
            // true boundaries: the walk up to the meeting point, the speculative marks from it on
            if (walker) {
                for (u32 x = 0; x < sw; x++) {
                    const u32 wi = (q0 >> 5) + x, base = wi * 32;
                    const u32 keep = !synced || meet >= base + 32 ? 0u : (meet <= base ? ~0u : ~0u << (meet - base));
                    S.bm[wi] = S.tm[wi] | (S.bm[wi] & keep);
                }
            }
            // symbols before each bitmap word (lanes own sw consecutive words)
            u32 own = 0;
            for (u32 x = 0; x < sw; x++) own += __popc(S.bm[lane * sw + x]);
            u32 o = own;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u32 v = __shfl_up_sync(FULL, o, d);
                if (lane >= d) o += v;
            }
            const u32 total = __shfl_sync(FULL, o, 31);
            const int ln = (int)((bl - 1) / seg);   // last lane with bits
            const u32 last = __shfl_sync(FULL, Eout, ln);
            o -= own;
            for (u32 x = 0; x < sw; x++) {
                S.wpre[lane * sw + x] = (u16)o;
                o += __popc(S.bm[lane * sw + x]);
            }
            bad = __any_sync(FULL, lbad) || total != (u32)vol || last != bl;
            __syncwarp();
            if (!bad) {
                // bit position of symbol index T: the largest word with wpre <= T, then its bit
                const u32 nbw = 32 * sw;
                auto select = [&](u32 T) -> u32 {
                    u32 lo = 0, hi = nbw;
                    while (hi - lo > 1) {
                        const u32 mid = (lo + hi) >> 1;
                        if (S.wpre[mid] <= T) lo = mid;
                        else hi = mid;
                    }
                    return lo * 32 + (u32)__fns(S.bm[lo], 0, (int)(T - S.wpre[lo]) + 1);
                };
                // row checkpoints for k_redecode: bit offset of every RD_SEG-th row start
                if (A.ckpt && lane >= 1 && lane <= RD_NCK && lane * RD_SEG < nrows)
                    A.ckpt[(size_t)b * RD_NCK + lane - 1] = select((u32)(lane * RD_SEG * bz));
                // ---- 3. symbols into the array: an equal share of codes per lane, two per look-up
                const u32 i0 = ((u32)lane * (u32)vol) >> 5, i1 = ((u32)(lane + 1) * (u32)vol) >> 5;
                if (i0 < i1) {
                    u32 pos = select(i0), i = i0;
                    while (i < i1) {
                        const u32 x = P0 + pos;
                        const u64 ent = lds_u64(tab_sa + 8u * (dw_win32(S.sb, x) >> (32 - PAIR_TBITS)));
                        if (((u32)ent & 0xc0u) == 0x80u && i + 1 < i1) {
                            S.sym[i] = (u16)(ent >> 16);
                            S.sym[i + 1] = (u16)(ent >> 32);
                            pos += (u32)ent & 63u;
                            i += 2;
                        } else {
                            u32 s0;
                            pos += (u32)dw_sym(S.sb, x, tab_sa, A.dsym, s0);
                            S.sym[i] = (u16)s0;
                            i++;
                        }
                    }
                }
            }
        } else {
            // ---- oversized slice: lane 0 decodes it alone from global memory
            if (lane == 0) {
                u32 pos = 0;
                for (int i = 0; i < vol && !bad; i++) {
                    const u32 x = P0 + pos;
                    u32 wv[3];
#pragma unroll
                    for (int q = 0; q < 3; q++) {
                        const u64 wi = w0 + (x >> 5) + q;
                        wv[q] = wi < bufw ? __byte_perm(__ldg(pay_words + wi), 0, 0x0123) : 0u;
                    }
                    const u32 s = x & 31;
                    const u64 w = ((u64)__funnelshift_l(wv[1], wv[0], s) << 32) | __funnelshift_l(wv[2], wv[1], s);
                    const u64 ent = ptab[(u32)(w >> (64 - PAIR_TBITS))];
                    u32 sym;
                    int l;
                    if ((u32)ent & 0xc0u) { sym = (u32)(ent >> 16) & 0xffffu; l = (int)(ent >> 8) & 63; }
                    else l = dw_long(w, A.dsym, sym);
                    if (!l) { bad = true; break; }
                    const int rr = i / bz;
                    if (A.ckpt && i % bz == 0 && rr && rr % RD_SEG == 0 && rr / RD_SEG <= RD_NCK)
                        A.ckpt[(size_t)b * RD_NCK + rr / RD_SEG - 1] = pos;
                    S.sym[i] = (u16)sym;
                    pos += (u32)l;
                    if (pos > bl && i + 1 < vol) bad = true;
                }
                if (pos != bl) bad = true;
            }
            bad = __shfl_sync(FULL, (int)bad, 0) != 0;
        }
        __syncwarp();
        if (bad) {
            if (lane == 0) fail_block(A, b, DF_PENDING, 0, 0);
            continue;
        }
        // ---- 4. reconstruction
        const u32 nunp = A.unpc[b];
        if (!recon) {
            // Lorenzo block: bins to scratch for k_recon_g; unpredictable count checked here
            u16* bins = A.bins + bins_index(g, b, 0);
            u32 zeros = 0;
            for (int p0 = 0; p0 < vol; p0 += 32) {
                const int p = p0 + lane;
                const u32 s = p < vol ? S.sym[p] : 1u;
                if (p < vol) bins[p] = (u16)s;
                zeros += __popc(__ballot_sync(FULL, s == 0u));
            }
            if (zeros != nunp && lane == 0) fail_block(A, b, DF_PENDING, 0, 0);
            __syncwarp();
            continue;
        }
        const float4 cf = load_coef(A.a, A.rec_off[b]);
        const double c0 = (double)cf.x, c1 = (double)cf.y, c2 = (double)cf.z, c3 = (double)cf.w;
        const u32 mby = 65535u / (u32)by + 1u;   // (r * mby) >> 16 == r / by for r < 2^16 / 9
        for (int r = lane; r < nrows; r += 32) {
            const int i = (int)(((u32)r * mby) >> 16), j = r - i * by;
            S.ab[r] = __dadd_rn(__dadd_rn(c0, __dmul_rn(c1, int_to_f64(i))), __dmul_rn(c2, int_to_f64(j)));
            S.rowoff[r] = (long long)i * plane + (long long)j * g.nz;
        }
        if (lane < bz) S.ck[lane] = __dmul_rn(c3, int_to_f64(lane));
        __syncwarp();
        float* obase = A.out + ((B.bi * DW_E) * g.ny + B.bj * DW_E) * g.nz + B.bk * DW_E;
        const u64 unp_base = A.info[DI_UNP_OFF] + 4 * A.uofs[b];
        u32 zeros = 0;
        u64 dsum = 0;
        // point p of the step is p0 + lane (row-major, so ballot order is point order)
        auto point = [&](bool in, int p, int r, int k, double ckk) {
            const u32 s = in ? S.sym[p] : 1u;
            float v = __double2float_rn(__dadd_rn(__dadd_rn(S.ab[r], ckk), __dmul_rn(twoeb, int_to_f64((int)s - center))));
            const unsigned zm = __ballot_sync(FULL, s == 0u);
            if (s == 0u) {
                const u32 zi = zeros + __popc(zm & ((1u << lane) - 1u));
                v = __uint_as_float(zi < nunp ? (u32)ld_le(A.a + unp_base + 4ull * zi, 4) : 0u);
            }
            zeros += __popc(zm);
            if (in) {
                dsum += (u64)__float_as_uint(v);
                obase[S.rowoff[r] + k] = v;
            }
        };
        if (bz == DW_E && nunp == 0) {
            // no unpredictable point (the common case): no ranks to form; a zero symbol is only
            // flagged (the count check below then fails the block)
            const int d = lane / DW_E, k = lane - d * DW_E;
            const double ckk = S.ck[k < bz ? k : 0];
            u32 z = 0;
            for (int r0 = 0; r0 < nrows; r0 += 3) {
                const int r = r0 + d;
                if (lane < 3 * DW_E && r < nrows) {
                    const u32 sy = S.sym[r * DW_E + k];
                    const float v = __double2float_rn(__dadd_rn(__dadd_rn(S.ab[r], ckk), __dmul_rn(twoeb, int_to_f64((int)sy - center))));
                    z |= sy == 0u;
                    dsum += (u64)__float_as_uint(v);
                    obase[S.rowoff[r] + k] = v;
                }
            }
            zeros = __popc(__ballot_sync(FULL, z != 0u));
        } else if (bz == DW_E) {
            // three rows of ten per step: lane = 10 d + k
            const int d = lane / DW_E, k = lane - d * DW_E;
            const double ckk = S.ck[k < bz ? k : 0];
            for (int r0 = 0; r0 < nrows; r0 += 3) {
                const int r = r0 + d;
                const bool in = lane < 3 * DW_E && r < nrows;
                point(in, in ? r * DW_E + k : 0, in ? r : 0, k, ckk);
            }
        } else {
            const u32 mbz = 65535u / (u32)bz + 1u;
            for (int p0 = 0; p0 < vol; p0 += 32) {
                const int p = p0 + lane;
                const bool in = p < vol;
                const int pp = in ? p : 0;
                const int r = (int)(((u32)pp * mbz) >> 16), k = pp - r * bz;
                point(in, pp, r, k, S.ck[k]);
            }
        }
        dsum = warp_sum_u64_redux(dsum);
        if (lane == 0) {
            if (zeros != nunp) fail_block(A, b, DF_PENDING, 0, 0);
            else if (has_sdc && stored_sum_dc(A, b) != dsum) {
                A.mflag[b] = 1;
                A.mis_list[atomicAdd(&A.counters[DC_NMIS], 1u)] = (u32)b;
            }
        }
        __syncwarp();
    }
}

}  // namespace ftlz
