// decompress.cu -- device side of container.parse (container.py:173-285) and
// pipeline.decompress (pipeline.py:645-723) for B200 (sm_100a).
//
// Kernel sequence:
//   k_parse_chunks   block table, speculative: for every 64-byte chunk and every entry phase
//                    (0..24) walk the variable-length records (9 or 25 bytes) -> exit phase;
//                    the chunk maps of each 256-chunk super-chunk composed in the same pass
//   k_parse_top      (> 256 super-chunks) threads the super-chunk maps from phase 0
//   k_parse_records  resolve every chunk's entry phase (with <= 256 super-chunks each CTA walks
//                    the super-chunk maps before its own), emit per-block records, validate
//   k_scan2          exclusive scans of bit lengths and unpredictable counts (look-back)
//   k_parse_tail     codebook + section validation, canonical code tables
//   k_dec_luts       the decode look-up tables, grid-wide
//   k_decode         lane = block: Huffman decode; regression blocks reconstructed in the
//                    same pass, staged in shared memory and written coalesced; Lorenzo bins to
//                    scratch; decompressed-data checksum verification (K6)
//   k_recon_warp     warp = block: Lorenzo wavefront reconstruction from scratch bins + verify;
//                    reused for re-execution of mismatching blocks (pipeline.py:713-723) (K7)
#include "common.cuh"

namespace ftlz {

#define PCHUNK 64
#define PSUPER 256
#define STUCK 0xffffffffu

enum {
    DI_TABLE_END = 0, DI_BOOK_OFF, DI_NSYM, DI_MAXLEN, DI_PAY_OFF, DI_PAY_LEN, DI_UNP_OFF,
    DI_NUNP, DI_SDC_OFF, DI_HAS_SDC, DI_TOTAL_BITS, DI_NREG, DI_T, DI_PAY_STORED, DI_SDC_STORED, DI_T12, DI_COUNT
};
enum { DC_NLOR = 0, DC_NMIS, DC_TICKET, DC_MINFAIL, DC_DTICKET, DC_COUNT };

struct DecArgs {
    Geom g;
    const u8* a;
    u64 len;
    int cap, center;
    double eb, twoeb;
    int codec;
    int n_faults;
    const ftlz_fault* faults;
    const int* fault_first;
    const ExtPlan* plans;
    const u32* coords;
    const u32* wave;
    const u32* wcrd;     // coordinates in wavefront order
    const u32* planes;
    u32* maps;
    u32* smaps;
    u64* sentry;
    long long nchunks, nsuper;
    // per block
    u8* ind;
    u64* rec_off;
    u32* unpc;
    u32* bitlen;
    u64* bofs;
    u64* uofs;
    u8* dflag;
    long long* da;
    long long* db;
    u8* mflag;
    u32* lor_list;
    u32* mis_list;
    u32* counters;
    u64* info;
    DevStatus* st;
    u32* lut;     // 2^T entries, T = min(maxlen, DEC_TBITS): the full-path decoder (one CTA per SM)
    u32* lut12;   // 2^T12 entries, T12 = min(maxlen, DEC_TBITS_S): list decodes with small CTAs
    u64* lut2;    // 2^14 two-symbol entries (decode_pairs.cu)
    u64* first_code;
    u32* lcount;
    u32* lbase;
    u32* dsym;
    u64* sortkeys;   // scratch for > 8192 symbols
    u16* bins;
    float* out;
    u32* lb_flag;
    u64* lb_a;
    u64* lb_b;
    // codec 1 (run-length): parse inverts the payload and the sum_dc section into these
    RleJob* rle_pay;
    RleJob* rle_sdc;
    u8* pay_scratch;
    u8* sdc_scratch;
    u64 pay_cap, sdc_cap;
    // region extraction (pipeline.py:726-795): output window in field coordinates
    int region;               // 1: k_decode list mode reports failures like the full path
    int list_spread;          // list mode: one block per warp (short lists: latency over lane use)
    u32* ckpt;                // full path: bit offset (in the block) of every RD_SEG-th row start, RD_NCK per block
    long long rx0, ry0, rz0, rnx, rny, rnz;
    const u32* region_list;   // the intersecting blocks, ascending
    u32 n_region;
    u32 pad_r2;
    // blocks [sb0, sb1) of the full path (k_decode, Lorenzo pass of k_recon_g): slabs of block
    // layers let the host download each finished slab while the next one decodes
    long long sb0, sb1;
};

FTLZ_DEV u64 ld_le(const u8* p, int n) {
    u64 v = 0;
    for (int i = 0; i < n; i++) v |= (u64)p[i] << (8 * i);
    return v;
}

// the payload the decoder reads (codec 0: inside the archive; codec 1: the inverted copy) and
// the byte offset of its first byte there; the raw sum_dc words likewise
FTLZ_DEV const u8* pay_base(const DecArgs& A) { return A.codec ? A.pay_scratch : A.a; }
FTLZ_DEV u64 pay_boff(const DecArgs& A) { return A.codec ? 0ull : A.info[DI_PAY_OFF]; }
FTLZ_DEV u64 stored_sum_dc(const DecArgs& A, long long b) {
    return ld_le((A.codec ? A.sdc_scratch : A.a + A.info[DI_SDC_OFF]) + 8ull * (u64)b, 8);
}

// ------------------------------------------------------------------------------------------
// block table parse (container.py:212-219)
// map value: exit phase (8 bits) | record count (24 bits); STUCK = error on this path.
// Walking chunk a then chunk b from entry phase s: map_apply(a, b, s).  Composition is
// associative, so the chunk and super-chunk walks are tree reductions / scans over maps.
FTLZ_DEV u32 map_apply(const u32* f, const u32* g, int s) {
    const u32 v = f[s];
    if (v == STUCK) return STUCK;
    const u32 w = g[v & 0xff];
    return w == STUCK ? STUCK : ((w & 0xff) | (((v >> 8) + (w >> 8)) << 8));
}

// entries of a walk from (st0, base0) through n <= 256 maps: entry[i] = (phase << 56 | record
// index) before map i, ~0 once the walk is stuck.  Two levels of 16 maps shorten the chain of
// dependent steps from n to <= 48: the 16-map group maps for all 25 phases, the walk over the
// groups, then every group's walk from its entry.  Returns the exit (STUCK or phase) and sets
// *base_out.  gm: 16 x 25 words, ge: 16 entries (shared).
#define WG 16
FTLZ_DEV u32 walk2(const u32* m, int n, u32 st0, u64 base0, u64* entry, u32* gm, u64* ge, u64* base_out) {
    const int ng = (n + WG - 1) / WG;
    for (int t = threadIdx.x; t < ng * 25; t += blockDim.x) {
        const int gi = t / 25, s = t - gi * 25;
        const int i1 = min(n, gi * WG + WG);
        u32 st = (u32)s, c = 0;
        for (int i = gi * WG; i < i1 && st != STUCK; i++) {
            const u32 v = m[i * 25 + st];
            st = v == STUCK ? STUCK : (v & 0xff);
            c += v == STUCK ? 0u : (v >> 8);
        }
        gm[t] = st == STUCK ? STUCK : (st | (c << 8));
    }
    __syncthreads();
    __shared__ u32 s_exit;
    __shared__ u64 s_base;
    if (threadIdx.x == 0) {
        u32 st = st0;
        u64 base = base0;
        for (int gi = 0; gi < ng; gi++) {
            ge[gi] = st == STUCK ? ~0ull : (((u64)st << 56) | base);
            if (st == STUCK) continue;
            const u32 v = gm[gi * 25 + st];
            st = v == STUCK ? STUCK : (v & 0xff);
            base += v == STUCK ? 0ull : (u64)(v >> 8);
        }
        s_exit = st;
        s_base = base;
    }
    __syncthreads();
    if ((int)threadIdx.x < ng) {
        const int gi = threadIdx.x;
        const u64 g0 = ge[gi];
        u32 st = g0 == ~0ull ? STUCK : (u32)(g0 >> 56);
        u64 base = g0 & ((1ull << 56) - 1);
        const int i1 = min(n, gi * WG + WG);
        for (int i = gi * WG; i < i1; i++) {
            entry[i] = st == STUCK ? ~0ull : (((u64)st << 56) | base);
            if (st == STUCK) continue;
            const u32 v = m[i * 25 + st];
            st = v == STUCK ? STUCK : (v & 0xff);
            base += v == STUCK ? 0ull : (u64)(v >> 8);
        }
    }
    __syncthreads();
    *base_out = s_base;
    return s_exit;
}

// chunk maps and their composition in one pass: the super-chunk's 256 chunks staged in shared
// memory (a walk never reads past its own chunk), each thread the 25 phase walks of one chunk
// (maps to global for k_parse_records), then the tree reduction to the super-chunk map
__global__ void __launch_bounds__(1024) k_parse_chunks(DecArgs A) {
    __shared__ u32 m[PSUPER * 25];
    __shared__ __align__(16) u8 sb[PSUPER * PCHUNK];
    const long long sc = blockIdx.x, c0 = sc * PSUPER;
    const int n = (int)min((long long)PSUPER, A.nchunks - c0);
    const u64 base = 55 + (u64)c0 * PCHUNK;
    // bytes past the archive read as 0xff: an indicator > 1 stops the walk like pos >= len
    for (int t = threadIdx.x; t < n * PCHUNK; t += blockDim.x) sb[t] = base + t < A.len ? A.a[base + t] : (u8)0xff;
    __syncthreads();
    // thread t: chunk t % 256, phases (t / 256) + 4 k
    const int ci = (int)threadIdx.x % PSUPER;
    if (ci < n) {
        const u8* cb = sb + ci * PCHUNK;
        for (int ph = (int)threadIdx.x / PSUPER; ph < 25; ph += 1024 / PSUPER) {
            int pos = ph;
            u32 cnt = 0;
            bool stuck = false;
            while (pos < PCHUNK) {
                const u8 ib = cb[pos];
                if (ib > 1) { stuck = true; break; }
                pos += 9 + 16 * ib;
                cnt++;
            }
            const u32 v = stuck ? STUCK : ((u32)(pos - PCHUNK) | (cnt << 8));
            m[ci * 25 + ph] = v;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n * 25; t += blockDim.x) A.maps[c0 * 25 + t] = m[t];
    for (int d = 1; d < n; d <<= 1) {
        const int np = (n - d + 2 * d - 1) / (2 * d);
        for (int t = threadIdx.x; t < np * 25; t += blockDim.x) {
            const int pi = t / 25, ss = t - pi * 25, i = pi * 2 * d;
            m[i * 25 + ss] = map_apply(m + i * 25, m + (i + d) * 25, ss);
        }
        __syncthreads();
    }
    if (threadIdx.x < 25) A.smaps[sc * 25 + threadIdx.x] = m[threadIdx.x];
}

// entry (phase, record index) of every super-chunk: the two-level walk over windows of 256
// super-chunk maps, the state carried between windows
__global__ void __launch_bounds__(256) k_parse_top(DecArgs A) {
    __shared__ u32 m[256 * 25];
    __shared__ u32 gm[WG * 25];
    __shared__ u64 ge[WG], ent[256];
    u32 st = 0;
    u64 base = 0;
    for (long long w0 = 0; w0 < A.nsuper; w0 += 256) {
        int n = (int)min(256ll, A.nsuper - w0);
        __syncthreads();
        for (int t = threadIdx.x; t < n * 25; t += blockDim.x) m[t] = A.smaps[w0 * 25 + t];
        __syncthreads();
        u64 nb;
        st = walk2(m, n, st, base, ent, gm, ge, &nb);
        base = nb;
        for (int i = threadIdx.x; i < n; i += blockDim.x) A.sentry[w0 + i] = ent[i];
    }
}

template <bool TOP>
__global__ void __launch_bounds__(PSUPER) k_parse_records(DecArgs A) {
    __shared__ u32 m[PSUPER * 25];
    __shared__ u32 gm[WG * 25];
    __shared__ u64 ge[WG], entry[PSUPER];
    long long sc = blockIdx.x;
    long long c0 = sc * PSUPER;
    int n = (int)min((long long)PSUPER, A.nchunks - c0);
    u64 se;
    if (TOP) {
        // (nsuper <= 256) this super-chunk's entry: the walk over the super-chunk maps before it
        if (sc == 0) se = 0;
        else {
            for (int t = threadIdx.x; t < (int)sc * 25; t += blockDim.x) m[t] = A.smaps[t];
            __syncthreads();
            u64 nb0;
            const u32 ex = walk2(m, (int)sc, 0, 0, entry, gm, ge, &nb0);
            se = ex == STUCK ? ~0ull : (((u64)ex << 56) | nb0);
            __syncthreads();
        }
    } else {
        se = A.sentry[sc];
    }
    if (se == ~0ull) return;
    for (int t = threadIdx.x; t < n * 25; t += blockDim.x) m[t] = A.maps[c0 * 25 + t];
    __syncthreads();
    u64 nb_unused;
    walk2(m, n, (u32)(se >> 56), se & ((1ull << 56) - 1), entry, gm, ge, &nb_unused);
    if ((int)threadIdx.x >= n) return;
    u64 en = entry[threadIdx.x];
    if (en == ~0ull) return;
    long long nb = A.g.nb;
    u64 s = 55 + (u64)(c0 + threadIdx.x) * PCHUNK, e = s + PCHUNK;
    u64 pos = s + (en >> 56);
    long long r = (long long)(en & ((1ull << 56) - 1));
    while (pos < e && r < nb) {
        if (pos + 1 > A.len) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, pos, -1, FTLZ_F_INDICATOR, 0, r); return; }
        u8 ib = A.a[pos];
        if (ib > 1) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_BAD_INDICATOR, pos, -1, ib, 0, r); return; }
        u64 q = pos + 1;
        if (ib) {
            if (q + 16 > A.len) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, q, -1, FTLZ_F_COEFFS, 0, r); return; }
            q += 16;
        }
        if (q + 8 > A.len) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, q, -1, FTLZ_F_RECORD, 0, r); return; }
        A.ind[r] = ib;
        A.rec_off[r] = pos;
        A.unpc[r] = (u32)ld_le(A.a + q, 4);
        A.bitlen[r] = (u32)ld_le(A.a + q + 4, 4);
        if (ib == 0) A.lor_list[atomicAdd(&A.counters[DC_NLOR], 1u)] = (u32)r;
        pos = q + 8;
        r++;
        if (r == nb) A.info[DI_TABLE_END] = pos;
    }
}

// ------------------------------------------------------------------------------------------
// exclusive scans of bitlen and unpc (u64) with decoupled look-back; tile = 1024 blocks
__global__ void __launch_bounds__(1024) k_scan2(DecArgs A) {
    if (dev_failed(A.st)) return;
    __shared__ u64 ws[2][32];
    __shared__ u64 pre[2];
    __shared__ unsigned s_tile;
    int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(&A.counters[DC_TICKET], 1u);
    __syncthreads();
    unsigned tile = s_tile;
    long long b = (long long)tile * 1024 + tid;
    bool v = b < A.g.nb;
    u64 x[2] = {v ? (u64)A.bitlen[b] : 0ull, v ? (u64)A.unpc[b] : 0ull};
    u64 inc[2];
#pragma unroll
    for (int q = 0; q < 2; q++) {
        inc[q] = x[q];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            u64 t = __shfl_up_sync(0xffffffffu, inc[q], o);
            if (lane >= o) inc[q] += t;
        }
        if (lane == 31) ws[q][warp] = inc[q];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < 2; q++) {
            u64 y = ws[q][lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                u64 t = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += t;
            }
            ws[q][lane] = y;   // inclusive over warps
        }
    }
    __syncthreads();
    if (warp == 0) {
        // look-back by the whole warp: lane l reads tile (t - l); the nearest tile holding an
        // inclusive prefix ends the walk, the aggregates before it are summed in one reduction
        volatile u64* va = A.lb_a; volatile u64* vb = A.lb_b; volatile u32* vf = A.lb_flag;
        u64 p0 = 0, p1 = 0;
        const u64 t0 = ws[0][31], t1 = ws[1][31];
        if (tile > 0) {
            if (lane == 0) {
                va[2 * tile] = t0; vb[2 * tile] = t1;
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
                if (zero & need) continue;   // a tile up to the stop has published nothing yet
                __threadfence();
                u64 a0 = 0, a1 = 0;
                if (lane < fi) { a0 = va[2 * ti]; a1 = vb[2 * ti]; }
                else if (lane == fi && f == 2u) { a0 = va[2 * ti + 1]; a1 = vb[2 * ti + 1]; }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
                    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
                }
                p0 += a0;
                p1 += a1;
                if (fi < 32) break;
                t -= 32;
            }
        }
        if (lane == 0) {
            va[2 * tile + 1] = p0 + t0; vb[2 * tile + 1] = p1 + t1;
            __threadfence();
            vf[tile] = 2;
            pre[0] = p0; pre[1] = p1;
            long long ntile = (A.g.nb + 1023) / 1024;
            if ((long long)tile == ntile - 1) {
                A.info[DI_TOTAL_BITS] = p0 + t0;
                A.info[DI_NUNP] = p1 + t1;
            }
        }
    }
    __syncthreads();
    if (v) {
        A.bofs[b] = pre[0] + (warp ? ws[0][warp - 1] : 0) + inc[0] - x[0];
        A.uofs[b] = pre[1] + (warp ? ws[1][warp - 1] : 0) + inc[1] - x[1];
    }
}

// ------------------------------------------------------------------------------------------
// codebook and sections (container.py:221-271) + canonical decode tables
#define PT_THREADS 1024
#define DEC_TBITS 15
#define DEC_TBITS_S 12

// phase 0: codec 0, everything.  Codec 1 runs three phases around the run-length inversions:
// 1 stops after the stored payload was taken (its job is filled), 2 checks the inverted payload
// and continues to the stored sum_dc section (its job is filled), 3 checks that inversion and
// finishes.  Every phase re-validates the codebook (cheap) so the positions are recomputed.
__global__ void __launch_bounds__(PT_THREADS) k_parse_tail(DecArgs A, int phase) {
    if (dev_failed(A.st)) return;
    extern __shared__ __align__(16) u64 pt_dyn[];  // 8192 keys
    __shared__ long long s_bad;
    __shared__ u64 s_kraft;
    __shared__ int s_maxlen;
    __shared__ u32 s_lc[64];
    __shared__ u64 s_fc[64];
    __shared__ u32 s_lb[64], s_pbase[64], s_pcnt[64 * (PT_THREADS / 32)];
    int tid = threadIdx.x;
    const u8* a = A.a;
    u64 len = A.len;
    u64 pos = A.info[DI_TABLE_END];
    if (tid == 0) { s_bad = -1; s_kraft = 0; s_maxlen = 0; }
    if (tid < 64) s_lc[tid] = 0;
    __syncthreads();
    if (pos + 4 > len) {
        if (tid == 0) dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, pos, -1, FTLZ_F_BOOK_SIZE, 0, 0);
        return;
    }
    u64 nsym = ld_le(a + pos, 4);
    pos += 4;
    u64 e0 = pos;
    u64 readable = (len - pos) / 5;   // entries fully inside the data
    u64 nchk = nsym < readable ? nsym : readable;
    // first failing entry in order (container.py:224-233)
    for (u64 t = tid; t < nchk; t += PT_THREADS) {
        const u8* ent = a + e0 + 5 * t;
        u64 sym = ld_le(ent, 4);
        int l = ent[4];
        bool bad = false;
        if (t > 0 && sym <= ld_le(ent - 5, 4)) bad = true;
        else if (sym >= (u64)A.cap) bad = true;
        else if (l < 1 || l > 57) bad = true;
        if (bad) atomicMin((unsigned long long*)&s_bad, (unsigned long long)t);
        else {
            atomicAdd(&s_lc[l], 1u);
            atomicMax(&s_maxlen, l);
        }
    }
    __syncthreads();
    long long bad = s_bad;
    if (bad >= 0 && (u64)bad < nchk) {
        if (tid == 0) {
            const u8* ent = a + e0 + 5 * (u64)bad;
            u64 sym = ld_le(ent, 4);
            int l = ent[4];
            u64 p = e0 + 5 * (u64)bad;
            if (bad > 0 && sym <= ld_le(ent - 5, 4)) dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_SYM_ORDER, p, -1, 0, 0, 0);
            else if (sym >= (u64)A.cap) dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_SYM_RANGE, p, -1, (long long)sym, 0, 0);
            else dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_BAD_LEN, p + 4, -1, l, 0, 0);
        }
        return;
    }
    if (nsym > readable) {
        if (tid == 0) dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, e0 + 5 * readable, -1, FTLZ_F_BOOK_ENTRY, 0, 0);
        return;
    }
    pos = e0 + 5 * nsym;
    if (tid == 0) {
        if (nsym == 0) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_EMPTY_BOOK, pos, -1, 0, 0, 0); return; }
        // Kraft: sum 2^(57-l) <= 2^57 (exact with per-length counts)
        unsigned __int128 k = 0;
        for (int l = 1; l <= 57; l++) k += (unsigned __int128)s_lc[l] << (57 - l);
        if (k > ((unsigned __int128)1 << 57)) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_KRAFT, pos, -1, 0, 0, 0); return; }
        if (pos + 8 > len) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, pos, -1, FTLZ_F_PAYLOAD_LEN, 0, 0); return; }
        u64 plen = ld_le(a + pos, 8);
        pos += 8;
        if (plen > len - pos) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, pos, -1, FTLZ_F_PAYLOAD, 0, 0); return; }
        if (A.codec != 0 && A.codec != 1) { dev_fail(A.st, FTLZ_ERR_UNSUPPORTED_CODEC, 0, -1, -1, A.codec, 0, 0); return; }
        u64 pay_off = pos;
        pos += plen;
        u64 dlen = plen;   // payload length after the backend inversion
        if (A.codec == 1) {
            if (phase == 1) {
                RleJob* J = A.rle_pay;
                J->in = a + pay_off; J->n = plen; J->out = A.pay_scratch; J->cap = A.pay_cap; J->flags = 0; J->out_len = 0;
                A.info[DI_PAY_OFF] = pay_off;
                A.info[DI_PAY_STORED] = plen;
                return;
            }
            const RleJob* J = A.rle_pay;
            if (J->flags & 1u) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_RLE_ODD, -1, -1, 0, 0, 0); return; }
            if (J->flags & 2u) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_RLE_ZERO, -1, -1, 0, 0, 0); return; }
            dlen = J->out_len;
        }
        u64 tb = A.info[DI_TOTAL_BITS];
        if (tb / 8 > dlen || (tb / 8 == dlen && (tb & 7))) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_BITS_EXCEED, pos, -1, 0, 0, 0); return; }
        if (A.codec == 1 && (tb + 7) / 8 + 8 > A.rle_pay->cap) {
            dev_fail(A.st, FTLZ_ERR_CAPACITY, 0, -1, -1, (long long)tb, 0, 0);
            return;
        }
        u64 nunp = A.info[DI_NUNP];
        if (nunp > (len - pos) / 4) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, pos, -1, FTLZ_F_UNPRED, 0, 0); return; }
        u64 unp_off = pos;
        pos += 4 * nunp;
        if (pos + 16 > len) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, pos, -1, FTLZ_F_SUMDC_LENS, 0, 0); return; }
        u64 raw = ld_le(a + pos, 8), stl = ld_le(a + pos + 8, 8);
        pos += 16;
        u64 nb = (u64)A.g.nb;
        if (raw != 0 && raw != 8 * nb) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_SUMDC_LEN, pos - 16, -1, (long long)raw, 0, 0); return; }
        u64 sdc_off = 0, has = 0;
        if (raw) {
            if (stl > len - pos) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRUNCATED, pos, -1, FTLZ_F_SUMDC, 0, 0); return; }
            sdc_off = pos;
            pos += stl;
            u64 rlen = stl;
            if (A.codec == 1) {
                if (phase == 2) {
                    RleJob* J = A.rle_sdc;
                    J->in = a + sdc_off; J->n = stl; J->out = A.sdc_scratch; J->cap = A.sdc_cap; J->flags = 0; J->out_len = 0;
                    return;
                }
                const RleJob* J = A.rle_sdc;
                if (J->flags & 1u) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_RLE_ODD, -1, -1, 0, 0, 0); return; }
                if (J->flags & 2u) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_RLE_ZERO, -1, -1, 0, 0, 0); return; }
                rlen = J->out_len;
            }
            if (rlen != raw) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_SUMDC_MISMATCH, pos, -1, 0, 0, 0); return; }
            has = 1;
        } else if (stl) {
            dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_ORPHAN, pos - 8, -1, 0, 0, 0);
            return;
        }
        if (A.codec == 1 && phase == 2) return;   // no sum_dc section to invert
        if (pos != len) { dev_fail(A.st, FTLZ_ERR_CORRUPT_STREAM, FTLZ_K_TRAILING, pos, -1, (long long)(len - pos), 0, 0); return; }
        A.info[DI_PAY_STORED] = plen;
        A.info[DI_SDC_STORED] = raw ? stl : 0;
        A.info[DI_BOOK_OFF] = e0 - 4;
        A.info[DI_NSYM] = nsym;
        A.info[DI_MAXLEN] = (u64)s_maxlen;
        A.info[DI_PAY_OFF] = pay_off;
        A.info[DI_PAY_LEN] = dlen;
        A.info[DI_UNP_OFF] = unp_off;
        A.info[DI_SDC_OFF] = sdc_off;
        A.info[DI_HAS_SDC] = has;
    }
    __syncthreads();
    if (dev_failed(A.st)) return;
    if (A.codec == 1 && phase != 3) return;
    // canonical order (length, symbol): symbols are strictly increasing already, so one stable
    // counting pass by length (cb_radix_pass) orders them
    const int n = (int)nsym;
    const bool small = n <= 4096;
    u64* keys = small ? pt_dyn : A.sortkeys;
    u64* sorted = small ? pt_dyn + 4096 : A.sortkeys + A.cap;
    for (int i = tid; i < n; i += PT_THREADS) {
        const u8* ent = a + e0 + 5 * (u64)i;
        keys[i] = ((u64)ent[4] << 32) | ld_le(ent, 4);
    }
    __syncthreads();
    cb_radix_pass<6>(keys, sorted, n, 32, s_pcnt, s_pbase);
    for (int i = tid; i < n; i += PT_THREADS) A.dsym[i] = (u32)(sorted[i] & 0xffffffffu);
    const int T = min(s_maxlen, DEC_TBITS);
    if (tid == 0) {
        u64 code = 0;
        u32 idx = 0;
        for (int l = 0; l < 64; l++) { A.first_code[l] = 0; A.lcount[l] = 0; A.lbase[l] = 0; }
        for (int l = 1; l <= 57; l++) {
            A.first_code[l] = code;
            A.lcount[l] = s_lc[l];
            A.lbase[l] = idx;
            s_fc[l] = code;
            s_lb[l] = idx;
            code = (code + s_lc[l]) << 1;
            idx += s_lc[l];
        }
        A.info[DI_T] = (u64)T;
        A.info[DI_T12] = (u64)min(s_maxlen, DEC_TBITS_S);
    }
    // (the decode LUTs are built by k_dec_luts over the whole grid)
}


// ------------------------------------------------------------------------------------------
// Huffman bit reader: MSB-first 64-bit window over the big-endian 32-bit words of one block's
// bit slice; positions are relative to the word holding the block's first bit (32-bit
// arithmetic).  Bits at or beyond `end` read as zero (the reference pads the slice with zero
// bytes, encode.py:214).  The next word is loaded one refill ahead so its latency overlaps
// decoding.
FTLZ_DEV u32 lds_u32(u32 addr) {
    u32 v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

struct BitReader {
    const u32* w;     // word 0: the word holding the block's first bit
    u32 endw;         // words [0, endw) are fully inside the slice
    u32 emask;        // valid-bit mask of word endw (0: none)
    u64 win;
    int have;
    u32 nw;           // index of the word held in `raw`
    u32 raw;          // raw (little-endian) word nw
};

FTLZ_DEV u32 br_word(const BitReader& R, u32 n, u32 raw) {
    const u32 v = __byte_perm(raw, 0, 0x0123);
    return n < R.endw ? v : (n == R.endw ? (v & R.emask) : 0u);
}
FTLZ_DEV u32 br_load(const BitReader& R, u32 n) { return n <= R.endw && (n < R.endw || R.emask) ? __ldg(R.w + n) : 0u; }

FTLZ_DEV void br_prefetch_ptr(const u32* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// L2 prefetch of the 128-byte line holding word n of the slice (no register, no scoreboard)
FTLZ_DEV void br_prefetch(const BitReader& R, u32 n) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(R.w + n));
}

// position the window at relative bit `pos`
FTLZ_DEV void br_seek(BitReader& R, u32 pos) {
    const u32 n = pos >> 5;
    R.win = ((u64)br_word(R, n, br_load(R, n)) << 32 | (u64)br_word(R, n + 1, br_load(R, n + 1))) << (pos & 31);
    R.have = 64 - (int)(pos & 31);
    R.nw = n + 2;
    if (R.have <= 32) {
        R.win |= (u64)br_word(R, R.nw, br_load(R, R.nw)) << (32 - R.have);
        R.have += 32;
        R.nw++;
    }
    R.raw = br_load(R, R.nw);
}

// slice [start, end) in absolute archive bits; returns the relative position of `start`
FTLZ_DEV u32 br_init(BitReader& R, const u8* a, u64 start, u64 end) {
    const u64 w0 = start >> 5;
    R.w = (const u32*)a + w0;
    const u64 rend = end > w0 * 32 ? end - w0 * 32 : 0;
    R.endw = (u32)(rend >> 5);
    R.emask = (rend & 31) ? (0xffffffffu << (32 - (u32)(rend & 31))) : 0u;
    const u32 pos = (u32)(start & 31);
    // the first lines of the slice go to L2 now; later lines are prefetched as the reader
    // crosses line boundaries (br_consume)
    for (u32 n = 32; n < 96u && n <= R.endw; n += 32) br_prefetch(R, n);
    br_seek(R, pos);
    return pos;
}

// predicated load: lanes with !p keep `v` (no divergent branch around the refill)
FTLZ_DEV u32 ldg_pred(const u32* ptr, bool p, u32 v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
        : "+r"(v)
        : "l"(ptr), "r"((u32)p));
    return v;
}

FTLZ_DEV void br_consume(BitReader& R, int l) {
    R.win <<= l;
    R.have -= l;
    const bool need = R.have <= 32;
    const u32 v = br_word(R, R.nw, R.raw);
    R.win |= need ? ((u64)v << (32 - R.have)) : 0ull;
    R.have += need ? 32 : 0;
    R.nw += need ? 1u : 0u;
    // next word (zero past the slice); a lane entering a new line prefetches two lines ahead
    const bool inside = R.nw <= R.endw && (R.nw < R.endw || R.emask);
    R.raw = ldg_pred(R.w + R.nw, need && inside, need ? 0u : R.raw);
    if (need && (R.nw & 31u) == 0u && R.nw + 64u <= R.endw) br_prefetch(R, R.nw + 64u);
}

// 64 bits at relative position pos (slow path)
FTLZ_DEV u64 br_peek64(const BitReader& R, u32 pos) {
    const u32 n = pos >> 5;
    const u64 hi = ((u64)br_word(R, n, br_load(R, n)) << 32) | br_word(R, n + 1, br_load(R, n + 1));
    const u32 w2 = br_word(R, n + 2, br_load(R, n + 2));
    const int sh = (int)(pos & 31);
    return sh ? ((hi << sh) | ((u64)w2 >> (32 - sh))) : hi;
}

// canonical decode tables of k_decode's slow path, at namespace scope so the path needs no
// registers for them across the symbol loop (k_decode fills them once per CTA)
__shared__ u64 s_dec_first[64];
__shared__ u32 s_dec_count[64], s_dec_base[64];
__shared__ int s_dec_T, s_dec_maxlen;

// a code longer than the table (or outside the code space: 0) at relative bit `cur`
FTLZ_DEV int decode_sym_slow(BitReader& R, const u32* dsym, u32 cur, u32* sym) {
    const u64 bits = br_peek64(R, cur);
    const int T = s_dec_T, maxlen = s_dec_maxlen;
    for (int l = T + 1; l <= maxlen; l++) {
        const u64 code = bits >> (64 - l);
        const u64 d = code - s_dec_first[l];
        if (d < (u64)s_dec_count[l]) {
            *sym = dsym[s_dec_base[l] + d];
            br_seek(R, cur + l);
            return l;
        }
    }
    return 0;
}

// ------------------------------------------------------------------------------------------
// Fast bit reader of the fault-free full path.  Same MSB-first window, but with no masking at
// the slice end: bits past the slice read as whatever the buffer holds (words past the buffer
// read as zero).  A block that decodes with consumed == bit_length, every code found and the
// right zero count had every code inside [start, start + bit_length), where both readers see
// the same bits, so its symbols equal the masked reader's; any other outcome is a failure of
// the masked reader too (contrapositive), and k_decode only marks such a block for the masked
// reader to classify (DF_PENDING).  Decompressed-data faults (FAULTS) change only the values
// written, never the decode.  Invariant after every refill: have >= 33.
struct FastReader {
    const u32* w;     // word 0: the word holding the block's first bit
    u32 lim;          // words [0, lim) may be loaded (the buffer's words, last one partial)
    u64 win;
    int have;
    u32 nw;           // index of the word held in `raw`
    u32 raw;          // raw (little-endian) word nw
};

FTLZ_DEV u32 fr_load(const FastReader& R, u32 n) { return n < R.lim ? __ldg(R.w + n) : 0u; }

FTLZ_DEV void fr_seek(FastReader& R, u32 pos) {
    const u32 n = pos >> 5;
    R.win = ((u64)__byte_perm(fr_load(R, n), 0, 0x0123) << 32 | (u64)__byte_perm(fr_load(R, n + 1), 0, 0x0123))
            << (pos & 31);
    R.have = 64 - (int)(pos & 31);
    R.nw = n + 2;
    if (R.have <= 32) {
        R.win |= (u64)__byte_perm(fr_load(R, R.nw), 0, 0x0123) << (32 - R.have);
        R.have += 32;
        R.nw++;
    }
    R.raw = fr_load(R, R.nw);
}

// relative bit position of the window's first bit
FTLZ_DEV u32 fr_pos(const FastReader& R) { return R.nw * 32u - (u32)R.have; }

// top up to >= 33 bits: one merge of the held word, one predicated load of the next
FTLZ_DEV void fr_refill(FastReader& R) {
    const bool need = R.have <= 32;
    const u32 v = need ? __byte_perm(R.raw, 0, 0x0123) : 0u;
    R.win |= (u64)v << ((32 - R.have) & 63);
    R.have += need ? 32 : 0;
    R.nw += need ? 1u : 0u;
    R.raw = ldg_pred(R.w + R.nw, need && R.nw < R.lim, need ? 0u : R.raw);
}

// one symbol with at least 12 bits in the window; a code longer than the table is searched in
// the window when the window holds maxlen bits (then topped up to >= 32 bits), else after a
// re-seek from the absolute position (>= 33 bits); returns false outside the code space
struct FrSlow {
    FastReader R;
    u32 sym, ok;
};
__device__ __noinline__ FrSlow fr_symbol_slow(FastReader R, const u32* dsym);

FTLZ_DEV bool fr_symbol(FastReader& R, u32 lut_sa, int lsh, const u32* dsym, u32& sym) {
    const u32 ent = lds_u32(lut_sa + 4u * (u32)(R.win >> lsh));
    if (ent) {
        const int l = (int)(ent & 63);
        sym = ent >> 8;
        R.win <<= l;
        R.have -= l;
        return true;
    }
    // a code longer than the table (rare): out of line, so the many inlined copies of the
    // symbol step stay small
    const FrSlow o = fr_symbol_slow(R, dsym);
    R = o.R;
    sym = o.sym;
    return o.ok != 0;
}

__device__ __noinline__ FrSlow fr_symbol_slow(FastReader R, const u32* dsym) {
    FrSlow o;
    o.ok = 0;
    o.sym = 0;
    u32& sym = o.sym;
    const int T = s_dec_T, maxlen = s_dec_maxlen;
    if (R.have >= maxlen) {
        // every code fits in the window's valid bits: search there, then top the window up
        for (int l = T + 1; l <= maxlen; l++) {
            const u64 d = (R.win >> (64 - l)) - s_dec_first[l];
            if (d < (u64)s_dec_count[l]) {
                sym = dsym[s_dec_base[l] + d];
                R.win <<= l;
                R.have -= l;
                fr_refill(R);
                o.ok = 1;
                o.R = R;
                return o;
            }
        }
        o.R = R;
        return o;
    }
    const u32 cur = fr_pos(R);
    const u32 n = cur >> 5;
    const u64 hi = ((u64)__byte_perm(fr_load(R, n), 0, 0x0123) << 32) | __byte_perm(fr_load(R, n + 1), 0, 0x0123);
    const u32 w2 = __byte_perm(fr_load(R, n + 2), 0, 0x0123);
    const int sh = (int)(cur & 31);
    const u64 bits = sh ? ((hi << sh) | ((u64)w2 >> (32 - sh))) : hi;
    for (int l = T + 1; l <= maxlen; l++) {
        const u64 code = bits >> (64 - l);
        const u64 d = code - s_dec_first[l];
        if (d < (u64)s_dec_count[l]) {
            sym = dsym[s_dec_base[l] + d];
            fr_seek(R, cur + l);
            o.ok = 1;
            o.R = R;
            return o;
        }
    }
    o.R = R;
    return o;
}

#define DF_PENDING 0xffu   // dflag: failed on the fast path, kind not yet classified
#define RD_SEG 10   // rows per re-decode segment
#define RD_NCK 9    // row checkpoints kept per block (segments 1..9 of 10)

FTLZ_DEV float4 load_coef(const u8* a, u64 rec) {
    const u8* p = a + rec + 1;
    float4 c;
    c.x = __uint_as_float((u32)ld_le(p, 4));
    c.y = __uint_as_float((u32)ld_le(p + 4, 4));
    c.z = __uint_as_float((u32)ld_le(p + 8, 4));
    c.w = __uint_as_float((u32)ld_le(p + 12, 4));
    return c;
}

FTLZ_DEV float apply_decomp_faults(const DecArgs& A, long long b, int p, int f0, float v) {
    for (int f = f0; f < A.n_faults && A.faults[f].block == b; f++)
        if (A.faults[f].target == FTLZ_FAULT_DECOMP && A.faults[f].element == p)
            v = __uint_as_float(__float_as_uint(v) ^ (1u << A.faults[f].bit));
    return v;
}

FTLZ_DEV void fail_block(const DecArgs& A, long long b, int kind, long long x, long long y) {
    A.dflag[b] = (u8)kind;
    A.da[b] = x;
    A.db[b] = y;
    atomicMin(&A.counters[DC_MINFAIL], (u32)b);
}

// ------------------------------------------------------------------------------------------
// K6: lane = block.  Warp = 32 consecutive blocks, decoded row by row in lockstep so that the
// warp's rows (contiguous along z for blocks of one block-row) are written coalesced.
#define DEC_WARPS 32   // one CTA per SM (64 registers x 1024 threads) sharing one decode table
// stage words per warp: 32 rows of e plus up to 3 words of alignment shift per run, 16-byte
// multiple
__host__ __device__ inline size_t dec_stage_words(int e) { return ((size_t)32 * e + 96 + 3) & ~(size_t)3; }
#define MAXE 64


template <bool FAULTS, bool FAST>
__global__ void __launch_bounds__(DEC_WARPS * 32, 1) k_decode(DecArgs A, const u32* list, int nlist) {
    if (dev_failed(A.st)) return;
    extern __shared__ __align__(16) unsigned char dsm[];
    const Geom& g = A.g;
    // list decodes (few blocks, small CTAs) stage the 12-bit table, the full path the 15-bit one
    const bool tsmall = list != nullptr;
    const int T = (int)A.info[tsmall ? DI_T12 : DI_T];
    const u32* lut_g = tsmall ? A.lut12 : A.lut;
    u32* s_lut = (u32*)dsm;
    float* stage_all = (float*)(dsm + ((size_t)4 << (tsmall ? DEC_TBITS_S : DEC_TBITS)));
    __shared__ long long s_rbase[DEC_WARPS][32];
    __shared__ int s_rlen[DEC_WARPS][32], s_rbx[DEC_WARPS][32], s_rby[DEC_WARPS][32], s_rpad[DEC_WARPS][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int x = tid; x < (1 << T); x += blockDim.x) s_lut[x] = lut_g[x];
    if (tid < 64) { s_dec_first[tid] = A.first_code[tid]; s_dec_count[tid] = A.lcount[tid]; s_dec_base[tid] = A.lbase[tid]; }
    if (tid == 0) { s_dec_T = T; s_dec_maxlen = (int)A.info[DI_MAXLEN]; }
    __syncthreads();
    u32 lut_sa;
    asm volatile("mov.u32 %0, %1;" : "=r"(lut_sa) : "r"(smem_u32(s_lut)));   // keep in a register
    const int lsh = 64 - T;
    float* stage = stage_all + (size_t)warp * dec_stage_words(g.e);
    const bool mode_list = list != nullptr;
    // one task: lane = block b (valid: b exists); every lane returns at the end of the task
    auto task = [&](const long long b, const bool valid) {
    const BlockInfo B = block_info(g, valid ? b : 0);
    const int kind = valid ? A.ind[b] : 0;
    const bool recon_here = valid && kind == 1 && !mode_list;
    const u64 pay_off = pay_boff(A), pay_len = A.info[DI_PAY_LEN];
    const u32 bl = valid ? A.bitlen[b] : 0;
    const u64 rel = valid ? A.bofs[b] : 0;
    int err = 0;
    long long ea = 0, eb2 = 0;
    const u64 last_byte = (rel + bl + 7) >> 3;
    if (valid && last_byte > pay_len) err = FTLZ_K_D_PAST_END;
    BitReader R;
    FastReader FR;
    const u64 start = pay_off * 8 + rel;
    u32 pos0;
    if constexpr (FAST) {
        const u64 s0 = valid && !err ? start : 0;
        const u64 w0 = s0 >> 5;
        const u64 bufw = ((A.codec ? A.pay_cap : A.len) + 3) >> 2;
        FR.w = (const u32*)pay_base(A) + w0;
        FR.lim = (u32)(bufw > w0 ? (bufw - w0 < 0xffffffffull ? bufw - w0 : 0xffffffffull) : 0ull);
        if (!(valid && !err)) FR.lim = 0;
        pos0 = (u32)(s0 & 31);
        for (u32 n = 32; n < 96u && n < FR.lim; n += 32) br_prefetch_ptr(FR.w + n);
        fr_seek(FR, pos0);
    } else {
        pos0 = br_init(R, pay_base(A), valid && !err ? start : 0, valid && !err ? (pay_off + last_byte) * 8 : 0);
    }
    u32 consumed = 0;
    u32 zeros = 0;
    const u32 nunp = valid ? A.unpc[b] : 0;
    const u64 unp_base = A.info[DI_UNP_OFF] + 4 * (valid ? A.uofs[b] : 0);
    const float4 cf = recon_here ? load_coef(A.a, A.rec_off[b]) : make_float4(0, 0, 0, 0);
    const double c0 = (double)cf.x, c1 = (double)cf.y, c2 = (double)cf.z, c3 = (double)cf.w;
    const double twoeb = A.twoeb;
    const int center = A.center;
    const int f0 = (A.n_faults && valid) ? A.fault_first[b] : -1;
    u64 dsum = 0;
    // runs: lanes of one block row with consecutive bk are contiguous in memory; each run is
    // written back row by row with coalesced stores (structure computed once)
    unsigned heads = 0;
    const int e = g.e;
    if (!mode_list) {
        const long long pbi = __shfl_up_sync(0xffffffffu, B.bi, 1), pbj = __shfl_up_sync(0xffffffffu, B.bj, 1);
        const long long pbk = __shfl_up_sync(0xffffffffu, B.bk, 1);
        const bool pv = __shfl_up_sync(0xffffffffu, valid, 1);
        const bool prev_same = lane > 0 && pv && valid && pbi == B.bi && pbj == B.bj && pbk + 1 == B.bk;
        heads = __ballot_sync(0xffffffffu, valid && !prev_same);
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        // last lane of my run: the lane before the next head (or the last valid lane)
        const unsigned later = heads & (lane == 31 ? 0u : (~0u << (lane + 1)));
        const int hn = later ? __ffs(later) - 1 : 32;
        const unsigned runm = vm & (hn == 32 ? ~0u : ((1u << hn) - 1u)) & ~((1u << lane) - 1u);
        const int last = runm ? 31 - __clz(runm) : lane;
        const int lbz = __shfl_sync(0xffffffffu, B.bz, last);
        if ((heads >> lane) & 1u) {
            s_rbase[warp][lane] = ((B.bi * e) * g.ny + B.bj * e) * g.nz + B.bk * e;
            s_rlen[warp][lane] = (last - lane) * e + lbz;
            s_rbx[warp][lane] = B.bx;
            s_rby[warp][lane] = B.by;
        }
        __syncwarp();
    }
    // 16-byte write-back: when every row start is congruent mod 4 floats to its block's first
    // row (nz % 4 == 0) each run's stage rows are shifted by 0..3 floats so that stage and
    // output share the alignment mod 16 bytes (P_h: cumulative shift up to run h)
    const bool vec = !mode_list && (g.nz & 3) == 0 && ((size_t)A.out & 15) == 0;
    int soff = lane * e;
    if (vec) {
        if (lane == 0) {
            int P = 0;
            unsigned hm = heads;
            while (hm) {
                const int h = __ffs(hm) - 1;
                hm &= hm - 1;
                P += (int)((s_rbase[warp][h] - (long long)(h * e + P)) & 3);
                s_rpad[warp][h] = P;
            }
        }
        __syncwarp();
        const unsigned mine = heads & ((2u << lane) - 1u);
        if (mine) soff += s_rpad[warp][31 - __clz(mine)];
    }
    u32 st_sa;
    asm volatile("mov.u32 %0, %1;" : "=r"(st_sa) : "r"(smem_u32(stage + soff)));   // keep in a register
    // warp-uniform row shapes of the fast path: all rows of 10 (unrolled pairs) or all even
    const bool rows10 = FAST && __all_sync(0xffffffffu, !valid || B.bz == 10);
    const bool rows_even = FAST && __all_sync(0xffffffffu, !valid || (B.bz & 1) == 0);
    int i = 0, j = 0;
    for (int r = 0; r < e * e; r++) {
        const bool act = valid && !err && i < B.bx && j < B.by;
        if (FAST && act && !mode_list && A.ckpt) {
            // row checkpoints for a parallel re-decode (k_redecode): every RD_SEG-th row start
            const int rr = i * B.by + j;
            if (rr && rr % RD_SEG == 0 && rr / RD_SEG <= RD_NCK) A.ckpt[(size_t)b * RD_NCK + rr / RD_SEG - 1] = consumed;
        }
        if (act) {
            // every lane stages one word per point: the reconstructed float (regression blocks
            // of the full path) or the bin (Lorenzo blocks, re-execution)
            double ab = 0.0, dk = 0.0;
            if (recon_here) ab = __dadd_rn(__dadd_rn(c0, __dmul_rn(c1, int_to_f64(i))), __dmul_rn(c2, int_to_f64(j)));
            auto emit = [&](u32 sym, int k) {
                const double pred = __dadd_rn(ab, __dmul_rn(c3, dk));
                dk = __dadd_rn(dk, 1.0);
                float v = __double2float_rn(__dadd_rn(pred, __dmul_rn(twoeb, int_to_f64((int)sym - center))));
                if (sym == 0u)
                    v = (recon_here && zeros < nunp) ? __uint_as_float((u32)ld_le(A.a + unp_base + 4ull * zeros, 4)) : 0.0f;
                if (FAULTS && f0 >= 0 && recon_here) v = apply_decomp_faults(A, b, (i * B.by + j) * B.bz + k, f0, v);
                const u32 word = recon_here ? __float_as_uint(v) : sym;
                dsum += recon_here ? (u64)word : 0ull;
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(st_sa + 4u * (u32)k), "r"(word) : "memory");
                zeros += sym == 0;
            };
            if constexpr (FAST) {
                // Unpredictable points (bin 0) are rare: the symbol loop only records them in
                // zmask, and a fix-up after the row puts the stored words in place (and
                // corrects dsum).  dsum and the word of Lorenzo lanes are left unselected: only
                // regression lanes use them.
                u32 zmask = 0;
                auto femit = [&](u32 sym, int k, double dkv) {
                    const double pred = __dadd_rn(ab, __dmul_rn(c3, dkv));
                    float v = __double2float_rn(__dadd_rn(pred, __dmul_rn(twoeb, int_to_f64((int)sym - center))));
                    if (FAULTS && f0 >= 0 && recon_here) v = apply_decomp_faults(A, b, (i * B.by + j) * B.bz + k, f0, v);
                    const u32 word = recon_here ? __float_as_uint(v) : sym;
                    dsum += (u64)word;
                    // no memory clobber: the stores may move within the row (the row ends with
                    // an explicit compiler barrier before the write-back reads)
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(st_sa + 4u * (u32)k), "r"(word));
                    zmask |= (u32)(sym == 0u) << k;
                };
                // symbol pairs: one refill per pair (>= 32 bits before, <= 24 consumed)
                auto fpair = [&](int k, double dk0, double dk1) -> bool {
                    u32 s0, s1;
                    if (!fr_symbol(FR, lut_sa, lsh, A.dsym, s0)) return false;
                    if (!fr_symbol(FR, lut_sa, lsh, A.dsym, s1)) return false;
                    fr_refill(FR);
                    femit(s0, k, dk0);
                    femit(s1, k + 1, dk1);
                    return true;
                };
                if ((FR.nw & 31u) == 0u && FR.nw + 64u < FR.lim) br_prefetch_ptr(FR.w + FR.nw + 64u);
                if (rows10) {
#pragma unroll
                    for (int k = 0; k < 10; k += 2)
                        if (!fpair(k, (double)k, (double)(k + 1))) { err = DF_PENDING; break; }
                } else if (rows_even) {
                    double dk2 = 0.0;
                    for (int k = 0; k < B.bz; k += 2) {
                        if (!fpair(k, dk2, __dadd_rn(dk2, 1.0))) { err = DF_PENDING; break; }
                        dk2 = __dadd_rn(dk2, 2.0);
                    }
                } else {
                    double dk1 = 0.0;
                    for (int k = 0; k < B.bz; k++) {
                        u32 s0;
                        if (!fr_symbol(FR, lut_sa, lsh, A.dsym, s0)) { err = DF_PENDING; break; }
                        fr_refill(FR);
                        femit(s0, k, dk1);
                        dk1 = __dadd_rn(dk1, 1.0);
                    }
                }
                asm volatile("" ::: "memory");
                while (zmask) {
                    const int k = __ffs(zmask) - 1;
                    zmask &= zmask - 1;
                    if (recon_here) {
                        u32 w = zeros < nunp ? (u32)ld_le(A.a + unp_base + 4ull * zeros, 4) : 0u;
                        if (FAULTS && f0 >= 0)
                            w = __float_as_uint(apply_decomp_faults(A, b, (i * B.by + j) * B.bz + k, f0, __uint_as_float(w)));
                        const u32 old = lds_u32(st_sa + 4u * (u32)k);
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(st_sa + 4u * (u32)k), "r"(w) : "memory");
                        dsum += (u64)w - (u64)old;
                    }
                    zeros++;
                }
                consumed = fr_pos(FR) - pos0;
            } else
            // The reference tests "ran past the slice" before every symbol.  Here it is tested
            // once per row (below) and before the slow path, the only place another error can
            // arise: symbols decoded past the slice are garbage of a block that fails anyway.
            for (int k = 0; k < B.bz; k++) {
                u32 ent = lds_u32(lut_sa + 4u * (u32)(R.win >> lsh));
                u32 sym;
                int l;
                if (ent) {
                    l = (int)(ent & 63);
                    sym = ent >> 8;
                    br_consume(R, l);
                } else {
                    if (consumed > bl) { err = FTLZ_K_D_RAN_PAST; break; }
                    l = decode_sym_slow(R, A.dsym, pos0 + consumed, &sym);
                    if (l == 0) { err = FTLZ_K_D_OUTSIDE; break; }
                }
                consumed += (u32)l;
                emit(sym, k);
            }
            // past the slice with symbols left (the last symbol's overrun is the reference's
            // consumed != bit_length check at the end)
            if (!err && consumed > bl && !(i == B.bx - 1 && j == B.by - 1)) err = FAST ? DF_PENDING : FTLZ_K_D_RAN_PAST;
        }
        __syncwarp();
        if (!mode_list) {
            const long long rowoff = ((long long)i * g.ny + j) * g.nz;
            unsigned hm = heads;
            while (hm) {
                const int h = __ffs(hm) - 1;
                hm &= hm - 1;
                if (i < s_rbx[warp][h] && j < s_rby[warp][h]) {
                    const int L = s_rlen[warp][h];
                    const long long base = s_rbase[warp][h] + rowoff;
                    if (vec) {
                        const float* src = stage + h * e + s_rpad[warp][h];
                        float* dst = A.out + base;
                        const int a0 = min((int)((-base) & 3), L);
                        const int n4 = (L - a0) >> 2, t0 = a0 + 4 * n4;
                        if (lane < a0) dst[lane] = src[lane];
                        if (lane < L - t0) dst[t0 + lane] = src[t0 + lane];
                        const float4* s4 = (const float4*)(src + a0);
                        float4* d4 = (float4*)(dst + a0);
                        for (int o = lane; o < n4; o += 32) d4[o] = s4[o];
                    } else {
                        for (int o = lane; o < L; o += 32) A.out[base + o] = stage[h * e + o];
                    }
                }
            }
        }
        if (act && !recon_here) {
            // bins of this row to scratch (Lorenzo blocks are reconstructed by k_recon_g, whose
            // output overwrites the run copy above)
            const u32* sw = (const u32*)stage + soff;
            const int pbase = (i * B.by + j) * B.bz;
            for (int k = 0; k < B.bz; k++) A.bins[bins_index(g, b, pbase + k)] = (u16)sw[k];
        }
        __syncwarp();
        if (++j == e) {
            j = 0;
            i++;
        }
    }
    if (valid && !err && consumed != bl) { err = FTLZ_K_D_CONSUMED; ea = (long long)consumed; eb2 = (long long)bl; }
    if (valid && !err && zeros != nunp) { err = FTLZ_K_D_ZEROS; ea = zeros; eb2 = nunp; }
    if (FAST && valid && err && err != FTLZ_K_D_PAST_END) err = DF_PENDING;   // classified by the masked reader
    if (valid && err) {
        if (mode_list && !A.region) A.mflag[b] = 3;
        else fail_block(A, b, err, ea, eb2);
        return;
    }
    if (recon_here && A.info[DI_HAS_SDC]) {
        const u64 stored = stored_sum_dc(A, b);
        if (stored != dsum) {
            A.mflag[b] = 1;
            A.mis_list[atomicAdd(&A.counters[DC_NMIS], 1u)] = (u32)b;
        }
    }
    };
    if (mode_list) {
        // re-execution: lane over the given block list, decode only (bins to scratch); a short
        // list spreads one block per warp (each block's decode is a serial chain: more warps,
        // shorter wall time, and no other lane's rows to write back)
        const long long wid = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
        const long long idx = A.list_spread ? wid : wid * 32 + lane;
        const bool valid = idx < (long long)nlist && (!A.list_spread || lane == 0);
        task(valid ? (long long)list[idx] : 0, valid);
        return;
    }
    // full path: warp task t = blocks sb0 + 32 t .. + 31.  One CTA per SM; CTA c takes the
    // tasks [c ntask / grid, (c + 1) ntask / grid), so every SM decodes the same number of
    // tasks (+-1): with one wave of CTAs of a few warps the SMs that received an extra CTA set
    // the kernel time
    const u32 ntask = (u32)((A.sb1 - A.sb0 + 31) / 32);
    const u32 t0 = (u32)((u64)blockIdx.x * ntask / gridDim.x), t1 = (u32)((u64)(blockIdx.x + 1) * ntask / gridDim.x);
    for (u32 t = t0 + warp; t < t1; t += blockDim.x >> 5) {
        const long long b = A.sb0 + (long long)t * 32 + lane;
        task(b < A.sb1 ? b : 0, b < A.sb1);
    }
}

// ------------------------------------------------------------------------------------------
// K6b / K7: warp = block reconstruction from scratch bins (both predictors), verification.
// mode 0: Lorenzo list, faults applied, mismatch -> mis_list.
// mode 1: re-execution of mis_list (no faults); verdict in mflag (2 ok, 3 still mismatching).
// G = threads per block group: 32 (a warp per block) or 128 (a CTA per block: the plane
// wavefront then covers a whole plane per step, which shortens the per-block latency chain)
// k_recon_g's per-group shared memory: float64 recon, float32 output, bins and, when it fits
// (block edges up to 20), the wavefront plan
__host__ __device__ inline bool recon_plan_fits(int vmax) { return vmax <= 8000; }
__host__ __device__ inline size_t recon_slot_bytes(int vmax, int nvmax8) {
    return (((size_t)vmax * 8 + 15) & ~(size_t)15) + (((size_t)vmax * 4 + 15) & ~(size_t)15) +
           (((size_t)nvmax8 * 2 + 15) & ~(size_t)15) + (recon_plan_fits(vmax) ? (((size_t)vmax * 4 + 4 * 80 + 15) & ~(size_t)15) : 0);
}

template <int G>
__global__ void __launch_bounds__(128) k_recon_g(DecArgs A, int mode) {
    if (dev_failed(A.st)) return;
    extern __shared__ __align__(16) unsigned char rsm[];
    const Geom& g = A.g;
    const int warp = threadIdx.x / G, lane = threadIdx.x % G;   // group, rank in group
    const int nw = blockDim.x / G;
    const int wl = threadIdx.x & 31, wi = (threadIdx.x % G) >> 5;   // lane / warp in the group
    __shared__ u64 s_red[4];
    __shared__ u32 s_cnt[4];
    auto gsync = [&]() {
        if (G == 32) __syncwarp();
        else __syncthreads();
    };
    // exclusive rank of `flag` among the group's ranks this step + the step's total
    auto gscan = [&](bool flag, u32& before, u32& total) {
        const unsigned m = __ballot_sync(0xffffffffu, flag);
        if (G == 32) {
            before = __popc(m & ((1u << wl) - 1u));
            total = __popc(m);
        } else {
            if (wl == 0) s_cnt[wi] = __popc(m);
            __syncthreads();
            u32 pre = 0, tot = 0;
            for (int q = 0; q < G / 32; q++) {
                if (q < wi) pre += s_cnt[q];
                tot += s_cnt[q];
            }
            __syncthreads();
            before = pre + __popc(m & ((1u << wl) - 1u));
            total = tot;
        }
    };
    auto gsum = [&](u64 v) -> u64 {
        v = warp_sum_u64(v);
        if (G == 32) return v;
        if (wl == 0) s_red[wi] = v;
        __syncthreads();
        u64 t = 0;
        for (int q = 0; q < G / 32; q++) t += s_red[q];
        __syncthreads();
        return t;
    };
    const size_t slot_bytes = recon_slot_bytes(g.vmax, g.nvmax8);
    double* xd = (double*)(rsm + (size_t)warp * slot_bytes);
    float* v32 = (float*)(xd + g.vmax);
    u16* sb = (u16*)(rsm + (size_t)warp * slot_bytes + (((size_t)g.vmax * 8 + 15) & ~(size_t)15) +
                     (((size_t)g.vmax * 4 + 15) & ~(size_t)15));
    // the wavefront plan of the group's current extent: (p << 32 | coords) in plane order, and the
    // plane starts (staged once per extent: the plane loop then reads no global memory)
    u32* wpc = (u32*)((unsigned char*)sb + (((size_t)g.nvmax8 * 2 + 15) & ~(size_t)15));   // p | i << 13 | j << 18 | k << 23
    int* wpl = (int*)(wpc + g.vmax);
    int plan_xid = -1;
    // mode 0: Lorenzo list; 1: re-execution list; 2: region list; 3: region re-execution
    const bool rgn = mode >= 2, reexec = mode & 1;
    u32 n = reexec ? A.counters[DC_NMIS] : (rgn ? A.n_region : A.counters[DC_NLOR]);
    const u32* list = reexec ? A.mis_list : (rgn ? A.region_list : A.lor_list);
    for (long long idx = (long long)blockIdx.x * nw + warp; idx < (long long)n; idx += (long long)gridDim.x * nw) {
        long long b = list[idx];
        if (mode == 0 && (b < A.sb0 || b >= A.sb1)) continue;   // another slab's block
        if (A.dflag[b]) continue;                       // undecodable: reported separately
        if (reexec && A.mflag[b] == 3) continue;        // re-decode failed
        BlockInfo B = block_info(g, b);
        int kind = A.ind[b];
        const ExtPlan& PL = A.plans[B.xid];
        const u32* crd = A.coords + PL.coord_off;
        int vol = B.vol, byz = B.by * B.bz, bz = B.bz;
        u64 unp_base = A.info[DI_UNP_OFF] + 4 * A.uofs[b];
        // raw words of unpredictable points in row-major order
        u32 zc = 0;
        for (int p0 = 0; p0 < vol; p0 += G) {
            int p = p0 + lane;
            u32 bin = p < vol ? A.bins[bins_index(g, b, p)] : 1u;
            u32 before, total;
            gscan(bin == 0, before, total);
            if (bin == 0) v32[p] = __uint_as_float((u32)ld_le(A.a + unp_base + 4ull * (zc + before), 4));
            zc += total;
        }
        gsync();
        if (kind == 1) {
            float4 cf = load_coef(A.a, A.rec_off[b]);
            double c0 = (double)cf.x, c1 = (double)cf.y, c2 = (double)cf.z, c3 = (double)cf.w;
            for (int p = lane; p < vol; p += G) {
                u32 bin = A.bins[bins_index(g, b, p)];
                if (bin) {
                    u32 c = __ldg(crd + p);
                    int i = c & 0xff, j = (c >> 8) & 0xff, k = c >> 16;
                    double pred = __dadd_rn(__dadd_rn(__dadd_rn(c0, __dmul_rn(c1, int_to_f64(i))), __dmul_rn(c2, int_to_f64(j))),
                                            __dmul_rn(c3, int_to_f64(k)));
                    v32[p] = __double2float_rn(__dadd_rn(pred, __dmul_rn(A.twoeb, int_to_f64((int)bin - A.center))));
                }
            }
        } else {
            const bool splan = recon_plan_fits(g.vmax);
            if (splan && B.xid != plan_xid) {
                const u32* wave = A.wave + PL.wave_off;
                const u32* wcrd = A.wcrd + PL.wave_off;
                const u32* planes = A.planes + PL.plane_off;
                for (int q = lane; q < vol; q += G) {
                    const u32 c = __ldg(wcrd + q);
                    wpc[q] = __ldg(wave + q) | ((c & 0xffu) << 13) | (((c >> 8) & 0xffu) << 18) | ((c >> 16) << 23);
                }
                for (int q = lane; q <= PL.nplanes; q += G) wpl[q] = (int)__ldg(planes + q);
                plan_xid = B.xid;
            }
            // the block's bins in shared memory (one coalesced burst instead of a dependent
            // global load per point and plane)
            {
                const uint4* src = (const uint4*)(A.bins + bins_index(g, b, 0));
                const int nch = (vol + 7) >> 3;
                for (int c = lane; c < nch; c += G) ((uint4*)sb)[c] = __ldg(src + c);
                gsync();
            }
            const u32* planes_g = A.planes + PL.plane_off;
            for (int s = 0; s < PL.nplanes; s++) {
                const int q0 = splan ? wpl[s] : (int)__ldg(planes_g + s), q1 = splan ? wpl[s + 1] : (int)__ldg(planes_g + s + 1);
                for (int q = q0 + lane; q < q1; q += G) {
                    int p, i, j, k;
                    if (splan) {
                        const u32 pc = wpc[q];
                        p = (int)(pc & 0x1fffu); i = (int)((pc >> 13) & 31u); j = (int)((pc >> 18) & 31u); k = (int)(pc >> 23);
                    } else {
                        p = (int)__ldg(A.wave + PL.wave_off + q);
                        const u32 c = __ldg(A.wcrd + PL.wave_off + q);
                        i = c & 0xff; j = (c >> 8) & 0xff; k = c >> 16;
                    }
                    u32 bin = sb[p];
                    float v;
                    if (bin) {
                        double d100 = i > 0 ? xd[p - byz] : 0.0;
                        double d010 = j > 0 ? xd[p - bz] : 0.0;
                        double d001 = k > 0 ? xd[p - 1] : 0.0;
                        double d110 = (i > 0 && j > 0) ? xd[p - byz - bz] : 0.0;
                        double d101 = (i > 0 && k > 0) ? xd[p - byz - 1] : 0.0;
                        double d011 = (j > 0 && k > 0) ? xd[p - bz - 1] : 0.0;
                        double d111 = (i > 0 && j > 0 && k > 0) ? xd[p - byz - bz - 1] : 0.0;
                        double pred = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(d100, d010), d001), -d110), -d101), -d011), d111);
                        v = __double2float_rn(__dadd_rn(pred, __dmul_rn(A.twoeb, int_to_f64((int)bin - A.center))));
                        v32[p] = v;
                    } else {
                        v = v32[p];
                    }
                    xd[p] = f32_to_f64(v);
                }
                gsync();
            }
        }
        gsync();
        int f0 = (!mode && A.n_faults) ? A.fault_first[b] : -1;
        u64 s = 0;
        long long base = ((B.bi * g.e) * g.ny + B.bj * g.e) * g.nz + B.bk * g.e;
        for (int p = lane; p < vol; p += G) {
            float v = v32[p];
            if (f0 >= 0) v = apply_decomp_faults(A, b, p, f0, v);
            s += __float_as_uint(v);
            int i = p / byz, rem = p - (p / byz) * byz;
            int j = rem / bz, k = rem - (rem / bz) * bz;
            if (rgn) {
                // the block's intersection with the region window
                const long long x = B.bi * g.e + i - A.rx0, y = B.bj * g.e + j - A.ry0, z = B.bk * g.e + k - A.rz0;
                if (x >= 0 && x < A.rnx && y >= 0 && y < A.rny && z >= 0 && z < A.rnz)
                    A.out[(x * A.rny + y) * A.rnz + z] = v;
            } else {
                A.out[base + ((long long)i * g.ny + j) * g.nz + k] = v;
            }
        }
        s = gsum(s);
        if (lane == 0) {
            bool has = A.info[DI_HAS_SDC] != 0;
            u64 stored = has ? stored_sum_dc(A, b) : 0;
            if (reexec) A.mflag[b] = (has && stored != s) ? 3 : 2;
            else if (has && stored != s) {
                A.mflag[b] = 1;
                A.mis_list[atomicAdd(&A.counters[DC_NMIS], 1u)] = (u32)b;
            }
        }
        gsync();
    }
}

// ------------------------------------------------------------------------------------------
// STAGE_DECOMP_BEFORE_VERIFY faults on regression blocks (pipeline.py:690, armed once): the
// fault-free decoder has already written and verified the block; flip the injected bits in the
// output, re-verify the block against its stored sum_dc (pipeline.py:692-707) and, on a
// mismatch, queue it for re-execution like the decoder would have.  Lorenzo blocks receive their
// faults inside k_recon_g (mode 0).  Warp per faulted block (fblk: distinct block ids).
__global__ void k_decomp_faults(DecArgs A, const u32* fblk, int nfb) {
    const Geom& g = A.g;
    const int lane = threadIdx.x & 31;
    const int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (w >= nfb) return;
    const long long b = fblk[w];
    if (A.ind[b] != 1 || A.dflag[b] != 0) return;
    const BlockInfo B = block_info(g, b);
    const long long base = ((B.bi * g.e) * g.ny + B.bj * g.e) * g.nz + B.bk * g.e;
    const int byz = B.by * B.bz;
    auto addr = [&](int p) {
        const int i = p / byz, rem = p - i * byz, j = rem / B.bz, k = rem - j * B.bz;
        return base + ((long long)i * g.ny + j) * g.nz + k;
    };
    if (lane == 0)
        for (int f = A.fault_first[b]; f >= 0 && f < A.n_faults && A.faults[f].block == b; f++)
            if (A.faults[f].target == FTLZ_FAULT_DECOMP) {
                float* o = A.out + addr((int)A.faults[f].element);
                *o = __uint_as_float(__float_as_uint(*o) ^ (1u << A.faults[f].bit));
            }
    __syncwarp();
    if (!A.info[DI_HAS_SDC]) return;
    u64 sum = 0;
    for (int p = lane; p < B.vol; p += 32) sum += (u64)__float_as_uint(A.out[addr(p)]);
    sum = warp_sum_u64(sum);
    if (lane == 0 && sum != stored_sum_dc(A, b) && A.mflag[b] != 1) {
        A.mflag[b] = 1;
        A.mis_list[atomicAdd(&A.counters[DC_NMIS], 1u)] = (u32)b;
    }
}

// Re-decode of one block per warp for re-execution (pipeline.py:713-723): the warp copies the
// block's bit slice from the archive into shared memory with coalesced loads, then one lane
// decodes it from there (the serial Huffman chain without global-memory latency) and writes
// the bins to scratch for k_recon_g (mode 1).  The first pass decoded the same bytes without
// error, so a failure here (impossible for an intact archive) is reported as a mismatch.
#define RD_WARPS 4
#define RD_MAXW 2048   // slice words staged per warp (a block of <= 1150 points at 57 bits)
FTLZ_DEV void redecode_block(const DecArgs& A, const long long b, const u32* s_lut, u32* sl, int T, int maxlen, int lane);

__global__ void __launch_bounds__(RD_WARPS * 32) k_redecode(DecArgs A, const u32* list, int n) {
    extern __shared__ __align__(16) unsigned char rsm[];
    u32* s_lut = (u32*)rsm;
    u32* slice_all = s_lut + (1 << DEC_TBITS_S);
    const Geom& g = A.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int T = (int)A.info[DI_T12], maxlen = (int)A.info[DI_MAXLEN];
    for (int x = tid; x < (1 << T); x += blockDim.x) s_lut[x] = A.lut12[x];
    if (tid < 64) { s_dec_first[tid] = A.first_code[tid]; s_dec_count[tid] = A.lcount[tid]; s_dec_base[tid] = A.lbase[tid]; }
    __syncthreads();
    // n < 0: the count is the device's mismatch counter (launched before the host knows it),
    // warps stride over the list
    const int cnt = n >= 0 ? n : (int)A.counters[DC_NMIS];
    for (int w = blockIdx.x * RD_WARPS + warp; w < cnt; w += (n >= 0 ? cnt : gridDim.x * RD_WARPS))
        redecode_block(A, list[w], s_lut, slice_all + (size_t)warp * RD_MAXW, T, maxlen, lane);
}

FTLZ_DEV void redecode_block(const DecArgs& A, const long long b, const u32* s_lut, u32* sl, int T, int maxlen, int lane) {
    const Geom& g = A.g;
    const BlockInfo B = block_info(g, b);
    const u32 bl = A.bitlen[b];
    const u64 start = pay_boff(A) * 8 + A.bofs[b];
    const u64 w0 = start >> 5;
    const u32 nwords = (u32)(((start + bl + 31) >> 5) - w0) + 2;   // + 2: the 64-bit window's tail
    if (nwords > RD_MAXW) {
        if (lane == 0) A.mflag[b] = 3;
        return;
    }
    const u64 bufw = ((A.codec ? A.pay_cap : A.len) + 3) >> 2;
    const u32* src = (const u32*)pay_base(A);
    for (u32 i = lane; i < nwords; i += 32) {
        const u64 wi = w0 + i;
        sl[i] = wi < bufw ? __byte_perm(__ldg(src + wi), 0, 0x0123) : 0u;   // big-endian words
    }
    __syncwarp();
    // segments of RD_SEG rows decoded in parallel from the checkpoints of the first pass (lane
    // s: rows [s RD_SEG, (s + 1) RD_SEG)); each must end exactly where the next begins
    const int rows = B.bx * B.by;
    int nseg = A.ckpt ? min((rows + RD_SEG - 1) / RD_SEG, RD_NCK + 1) : 1;
    if (nseg > 1 && nseg * RD_SEG < rows) nseg = 1;   // more rows than checkpoints cover
    const u32 base = (u32)(start & 31);
    u32 sb = 0, se = bl;
    if (lane < nseg) {
        if (lane > 0) sb = A.ckpt[(size_t)b * RD_NCK + lane - 1];
        if (lane < nseg - 1) se = A.ckpt[(size_t)b * RD_NCK + lane];
    }
    const int p_lo = lane * RD_SEG * B.bz, p_hi = nseg == 1 ? B.vol : min((lane + 1) * RD_SEG * B.bz, B.vol);
    u32 pos = base + sb, zeros = 0;
    const u32 end = base + se;
    bool bad = sb > se || se > bl;
    if (lane < nseg && !bad) {
        for (int p = p_lo; p < p_hi; p++) {
            const u32 wi = pos >> 5, sh = pos & 31;
            const u64 hi = ((u64)sl[wi] << 32) | sl[wi + 1];
            const u64 win = sh ? (hi << sh) | ((u64)sl[wi + 2] >> (32 - sh)) : hi;
            const u32 ent = s_lut[(u32)(win >> (64 - T))];
            u32 sym = 0, l;
            if (ent) {
                l = ent & 63;
                sym = ent >> 8;
            } else {
                l = 0;
                for (int t = T + 1; t <= maxlen; t++) {
                    const u64 d = (win >> (64 - t)) - s_dec_first[t];
                    if (d < (u64)s_dec_count[t]) {
                        l = (u32)t;
                        sym = A.dsym[s_dec_base[t] + d];
                        break;
                    }
                }
                if (!l) { bad = true; break; }
            }
            pos += l;
            if (pos > end) { bad = true; break; }
            zeros += sym == 0u;
            A.bins[bins_index(g, b, p)] = (u16)sym;
        }
        bad |= pos != end;
    }
    const bool anybad = __any_sync(0xffffffffu, lane < nseg && bad);
    const u32 ztot = __reduce_add_sync(0xffffffffu, lane < nseg ? zeros : 0u);
    if (lane == 0 && (anybad || ztot != A.unpc[b])) A.mflag[b] = 3;
}

// verdicts of the re-executed blocks, in list order (2: matches after re-execution, else 3)
__global__ void k_reexec_verdict(DecArgs A, u8* verdict, int n) {
    const u32 cnt = n >= 0 ? (u32)n : A.counters[DC_NMIS];
    for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
        verdict[i] = A.mflag[A.mis_list[i]];
}

}  // namespace ftlz
