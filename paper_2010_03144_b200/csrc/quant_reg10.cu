// quant_reg10.cu -- stage (c) of pipeline.compress for regression blocks whose z rows hold 10
// points (the default block edge; pipeline.py:390-453, quantize.py:37-52, duplicated
// evaluation pipeline.py:157-179), one lane per pair of consecutive points of a z row.
//
// Decision in float32, reconstruction in float64.  The bin of a point is RN(S) with
// S = (x - p) / (2 eb) unless S lies at a half-integer (quantize.py: floor(|h| + 0.5) with the
// sign of diff), so the kernel estimates S in float32,
//     s = fma(x, rcp32, -fma(b3r, k, abr)),   abr = (ab / 2eb)_32, b3r = (b3 / 2eb)_32,
// whose distance to S is bounded by delta = 2^-21 |s| + 2^-20 (|abr| + 9 |b3r|) + 2^-40 (at least
// twice the worst-case float32 rounding, derivation in DESIGN.md section 4).  A point whose s
// lies within delta of a half-integer is flagged; every other point's bin is exact.  Points
// with |s| >= sbig (NaN, inf, far outliers) are unpredictable whatever their exact S.  The
// reconstruction pred + (2 eb)(bin - C) and the bin / float32 recon are then evaluated in
// float64 in the reference order (-fmad=false), and |x - recon32| <= eb is decided in float32
// with a 2^-20 relative guard band around eb (flagged inside it).  Duplicated evaluation
// recomputes the prediction from independently loaded coefficients and the reconstruction
// from its own 2 eb copy; any bit difference flags the point.  Flagged points (rare) are
// recomputed by the reference formulation (blocks.cu quant_point) in a per-lane fix-up, which
// also applies injected STAGE_DUP_EVAL faults.
//
// Layout: warp-autonomous persistent CTAs, each warp streams its regression blocks through
// two TMA tiles (tma.cuh); row r's ten points form pairs 5 r .. 5 r + 4 and lane l
// takes pairs l, l + 32, ... (500 pairs on a 10^3 block: 98% of the lane slots busy, against 78%
// for one lane per row).  The per-row terms (row prediction, its float32 scaled copy) are built
// once per block in shared memory (r10_rowtab).  A pair's two floats arrive in one 8-byte load,
// its bins leave as one 32-bit store straight into the encoder's bins array.  Histogram:
// lane-private u8 counters for the 128 bins around the centre (flushed every few blocks),
// out-of-window bins counted by a rescan of the lane's pairs.
namespace ftlz {

#ifndef R10_WARPS
#define R10_WARPS 12
#endif
#define R10_LH 128   // lane-private histogram window (bins center - 64 .. center + 63) + a sink row
#define R10_ROWS 100 // rows of a block (edge 10)

struct R10Acc {
    u32 bs;        // sum of bins
    u32 bis;       // sum of p * bin (a lane's <= 34 points of a block: < 2^32)
    u64 dc;        // sum of recon32 words
    u64 cs, csi;   // input checksum pair
    float emax;    // the lane's largest distance bound to a half-integer
    float amin;    // the lane's smallest | |x - recon32| - eb |
    u32 macc;      // OR of the duplicated evaluation's bit differences
    bool nz;       // some point of the lane is unpredictable
    FTLZ_DEV void reset() {
        bs = 0; bis = 0; dc = 0; cs = 0; csi = 0;
        emax = 0.0f; amin = INFINITY; macc = 0; nz = false;
    }
};

// lane-private u8 counters: bin o of the window in byte o & 3 of word (o >> 2) * 32 + lane, so
// every lane's counters sit in its own bank (no conflicts whatever the bins).  A bin outside the
// window only bumps the lane's sink counter (word row R10_LH / 4): no branch in the point loop;
// when the sink moved, the lane's bins are recounted afterwards into the CTA's shared window
// (hwin, HWIN_REG bins) or, beyond it, the global histogram.
#define R10_LHBYTES ((R10_LH / 4 + 1) * 32 * 4)
struct R10Hist {
    unsigned char* lhw;   // this lane's column: lh + 4 lane
    u32* hwin;            // CTA window
    u64* ghist;
    int lhlo, wlo;
    FTLZ_DEV unsigned char* at(u32 o) const { return lhw + (o * 32u - (o & 3u) * 31u); }   // (o >> 2) 128 + (o & 3)
    // count `delta` (+1 / -1) for bin b (slow paths: fix-up, recount, undo)
    FTLZ_DEV void add(u32 b, int delta) const {
        const u32 o = b - (u32)lhlo;
        if (o < (u32)R10_LH) *at(o) += (unsigned char)delta;
        else reg_hist_out(hwin, ghist, wlo, (int)b, delta);
    }
    // hot path: window counter, or the sink for an out-of-window bin (recounted per block)
    FTLZ_DEV void bump(u32 b) const { *at(min(b - (u32)lhlo, (u32)R10_LH)) += 1; }
    FTLZ_DEV u32 sink() const { return *at(R10_LH); }
    FTLZ_DEV void set_sink(u32 v) const { *at(R10_LH) = (unsigned char)v; }
};

// lane l adds word row l (bins 4 l .. 4 l + 3) over the 32 lanes' words (rotated: conflict-free)
// into the global histogram and clears it
FTLZ_DEV void lh_flush10(u32* lh, u64* ghist, int lhlo, int cap, int lane) {
    static_assert(R10_LH == 128, "one word row per lane");
    __syncwarp();
    u32 se = 0, so = 0;   // bytes 0, 2 / 1, 3 of the words as 16-bit sums (<= 32 * 255)
#pragma unroll 8
    for (int c = 0; c < 32; c++) {
        u32* w = lh + lane * 32 + ((c + lane) & 31);
        const u32 v = *w;
        se += v & 0x00ff00ffu;
        so += (v >> 8) & 0x00ff00ffu;
        *w = 0;
    }
    const u32 sums[4] = {se & 0xffffu, so & 0xffffu, se >> 16, so >> 16};
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int bn = lhlo + 4 * lane + q;
        if (sums[q] && bn >= 0 && bn < cap) atomicAdd(&ghist[bn], (u64)sums[q]);
    }
    __syncwarp();
}

// per-row terms of a block, built once per block in the warp's shared-memory slot: the row
// prediction ((b0 + b1 i) + b2 j) (and its duplicate from the independently loaded
// coefficients), its float32 scaled copy and guard width, the row's tile offset
struct R10Row {
    double ab, ab2;
    float abr, erow;
    u32 toff;
    int ij;   // i << 16 | j
};

// a block's global operands, staged one block ahead (k_quant_reg10)
struct R10Pre {
    float4 cf, cg;    // coefficients; the duplicate's own copy
    u64 ins, inis;    // stage (a) checksum pair
    u32 nxt, pad[3];  // list entry after the next block (~0: none)
};

// one point of the fast path (see the file header): k is the lane's constant z offset, so
// ck = b3 k (and its duplicate ckd = b3' k) are per-lane constants; returns the bin (0:
// unpredictable) and the recon32 word, folds the flag terms into the lane's accumulators
template <bool DUP>
FTLZ_DEV u32 r10_point(const QuantParams& Q, float x, float kf, double ck, double ckd, const R10Row& R, float b3r,
                       u32 cbin, const R10Hist& H, R10Acc& acc, u32& rbits) {
    // float32 estimate of S and its distance to the nearest half-integer
    const float c = __fmaf_rn(b3r, kf, R.abr);
    const float s = __fmaf_rn(x, Q.rcp32, -c);
    const float m = __fadd_rn(s, 12582912.0f);   // 1.5 * 2^23: low mantissa bits = RN(s)
    const float f = __fadd_rn(s, -__fadd_rn(m, -12582912.0f));
    const bool big = !(fabsf(s) < Q.sbig);
    acc.emax = fmaxf(acc.emax, big ? 0.0f : __fadd_rn(fabsf(f), __fmaf_rn(fabsf(s), 4.76837158203125e-07f, R.erow)));
    const u32 bin = __float_as_uint(m) + cbin;
    const bool ok = !big && (bin - 1u) < (u32)(Q.cap - 1);
    // float64 reconstruction in the reference order
    const double offs = __int2double_rn((int)(__float_as_uint(m) - 0x4B400000u));
    const double p1 = __dadd_rn(R.ab, ck);
    const double d1 = __dadd_rn(p1, __dmul_rn(Q.twoeb, offs));
    if (DUP) {
        const double p2 = __dadd_rn(R.ab2, ckd);
        const double d2 = __dadd_rn(p2, __dmul_rn(Q.twoeb_dup, offs));
        const u64 xp = dbits(p1) ^ dbits(p2), xd = dbits(d1) ^ dbits(d2);
        acc.macc |= (u32)xp | (u32)(xp >> 32) | (u32)xd | (u32)(xd >> 32);
    }
    const float d32 = __double2float_rn(d1);
    const float a = __fadd_rn(fabsf(__fadd_rn(x, -d32)), -Q.eb32);
    acc.amin = fminf(acc.amin, ok ? fabsf(a) : INFINITY);
    const bool keep = ok && a <= 0.0f;
    acc.nz |= !keep;
    rbits = __float_as_uint(keep ? d32 : x);
    const u32 b = keep ? bin : 0u;
    H.bump(b);
    return b;
}

// exact recomputation of one point (reference formulation, blocks.cu quant_point) when its fast
// evaluation is flagged or it carries an injected duplicated-evaluation fault: replaces the
// fast results (bin, sums, histogram)
template <bool DUP>
FTLZ_DEV void r10_fix_point(const CompArgs& A, long long b, bool hasdup, const QuantParams& Q, float x, int p, int k,
                            double ab, double ab2, float abr, float erow, float b3r, double di, double dj,
                            const float4& cf, const float4& cg, u16* gbins, const R10Hist& H, R10Acc& acc,
                            bool& mism) {
    const double kd = int_to_f64(k);
    const double ckk = __dmul_rn((double)cf.w, kd), ck2k = DUP ? __dmul_rn((double)cg.w, kd) : ckk;
    // the fast path's result for this point (recomputed: same operations)
    const float c = __fmaf_rn(b3r, (float)k, abr);
    const float s = __fmaf_rn(x, Q.rcp32, -c);
    const float m = __fadd_rn(s, 12582912.0f);
    const float rr = __fadd_rn(m, -12582912.0f);
    const float f = __fadd_rn(s, -rr);
    const float dl = __fmaf_rn(fabsf(s), 4.76837158203125e-07f, erow);
    const bool big = !(fabsf(s) < Q.sbig);
    const int qi = (int)__float_as_uint(m) - 0x4B400000;
    const bool edge = !big && __fadd_rn(fabsf(f), dl) >= 0.49999905f;
    const u32 bin = (u32)(Q.center + qi);
    const bool ok = !big && (bin - 1u) < (u32)(Q.cap - 1);
    const double offs = int_to_f64(qi);
    const double p1 = __dadd_rn(ab, ckk);
    const double d1 = __dadd_rn(p1, __dmul_rn(Q.twoeb, offs));
    bool mis = false;
    if (DUP) {
        const double p2 = __dadd_rn(ab2, ck2k);
        const double d2 = __dadd_rn(p2, __dmul_rn(Q.twoeb_dup, offs));
        mis = dbits(p1) != dbits(p2) || dbits(d1) != dbits(d2);
    }
    const float d32 = __double2float_rn(d1);
    const float a = __fadd_rn(fabsf(__fadd_rn(x, -d32)), -Q.eb32);
    const bool unsure = ok && fabsf(a) <= Q.band32;
    const bool keep = ok && a <= 0.0f;
    const u32 fb = keep ? bin : 0u;
    const float rf = keep ? d32 : x;
    DupMask M;
    const bool fp = hasdup && dup_masks(A, b, p, M);
    if (!(edge || unsure || mis || fp || !Q.fast32)) return;
    if (!fp) {
#pragma unroll
        for (int q = 0; q < 3; q++) M.p[q] = M.r[q] = 0ull;
    }
    float rx;
    double back;
    const u32 ex = (u32)quant_point(
        Q, x, p1, DUP, [&] { return __dadd_rn(opaque(ab2), opaque(ck2k)); },
        [&] {
            return __dadd_rn(__dadd_rn(__dadd_rn((double)cf.x, __dmul_rn((double)cf.y, di)), __dmul_rn((double)cf.z, dj)),
                             __dmul_rn(opaque((double)cf.w), int_to_f64(k)));
        },
        M, &rx, &mism, &back);
    gbins[p] = (u16)ex;
    acc.bs += ex - fb;
    acc.bis += (u32)p * ex - (u32)p * fb;
    acc.dc += (u64)__float_as_uint(rx) - (u64)__float_as_uint(rf);
    if (ex == 0u) acc.nz = true;
    // drop the fast bin's count, count the exact bin
    H.add(fb, -1);
    H.add(ex, 1);
}

template <bool DUP>
FTLZ_DEV void r10_rowtab(R10Row* rt, int rows, int by, int tye, int tz, int zoff, const float4& cf, const float4& cg,
                         float b3r, double rcp32d, int lane) {
    const u32 m16 = 65535u / (u32)by + 1u;   // ceil(2^16 / by): (r m16) >> 16 = r / by for r < 2^16 / 9
    for (int r = lane; r < rows; r += 32) {
        const int i = (int)(((u32)r * m16) >> 16), j = r - i * by;
        const double di = int_to_f64(i), dj = int_to_f64(j);
        R10Row t;
        t.ab = __dadd_rn(__dadd_rn((double)cf.x, __dmul_rn((double)cf.y, di)), __dmul_rn((double)cf.z, dj));
        t.ab2 = DUP ? __dadd_rn(__dadd_rn((double)cg.x, __dmul_rn((double)cg.y, di)), __dmul_rn((double)cg.z, dj)) : t.ab;
        t.abr = __double2float_rn(__dmul_rn(t.ab, rcp32d));
        t.erow = __fmaf_rn(9.0f, fabsf(b3r), fabsf(t.abr)) * 9.5367431640625e-07f + 9.094947017729282e-13f;
        t.toff = (u32)((i * tye + j) * tz + zoff);
        t.ij = (i << 16) | j;
        rt[r] = t;
    }
    __syncwarp();
}

// compaction of the regression blocks after k_prep: 10-point-row blocks for k_quant_reg10
// (counters[5] entries of r10_list), the rest for k_quant_reg (counters[6], regx_list).  One
// atomic per CTA; list order is irrelevant (blocks are independent).
__global__ void __launch_bounds__(1024) k_reglist(CompArgs A) {
    __shared__ u32 wc[2][32];
    __shared__ u32 base[2];
    const Geom& g = A.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long b = (long long)blockIdx.x * 1024 + tid;
    bool reg = b < g.nb && A.ind[b] == 1 && !(A.events[b] & 4);
    bool q10 = false;
    if (reg && A.r10) {
        long long bi, bj, bk;
        block_coords(g, b, &bi, &bj, &bk);
        q10 = bk != g.cz - 1 || g.rz == 10;
    }
    const bool qx = reg && !q10;
    const unsigned m10 = __ballot_sync(0xffffffffu, q10), mx = __ballot_sync(0xffffffffu, qx);
    if (lane == 0) { wc[0][warp] = __popc(m10); wc[1][warp] = __popc(mx); }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const u32 v = wc[q][lane];
            u32 inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            wc[q][lane] = inc - v;
            if (lane == 31) base[q] = inc ? atomicAdd(&A.counters[5 + q], inc) : 0u;
        }
    }
    __syncthreads();
    if (q10) A.r10_list[base[0] + wc[0][warp] + __popc(m10 & ((1u << lane) - 1u))] = (u32)b;
    if (qx) A.regx_list[base[1] + wc[1][warp] + __popc(mx & ((1u << lane) - 1u))] = (u32)b;
}

#ifndef R10_MAXREG
#define R10_MAXREG (65536 / (R10_WARPS * 32) / 8 * 8)
#endif
template <bool DUP, bool PIN>
__global__ void __maxnreg__(R10_MAXREG) k_quant_reg10(const __grid_constant__ CompArgs A,
                                                                  const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const Geom& g = A.g;
    if (dev_failed(A.st)) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const StageCfg S = A.stage;
    unsigned char* slot = smem + (size_t)warp * A.r10_slot;
    WarpStager ws;
    ws.base = slot;
    ws.tbytes = S.tile_bytes;
    // slot: tile 0 | tile 1 | row table | lane counters | operands | mbarriers (tile 1 and the row
    // table are contiguous: the float64 buffer of the Lorenzo phase)
    R10Row* rowtab = (R10Row*)(slot + 2 * S.tile_bytes);   // R10_ROWS rows of the current block
    u32* lh = (u32*)(rowtab + R10_ROWS);                  // R10_LHBYTES of lane counters
    R10Pre* pre = (R10Pre*)((unsigned char*)lh + R10_LHBYTES);   // operands of the current / next block
    ws.bar = (u64*)(pre + 2);
    u32* hwin = (u32*)(smem + (size_t)nw * A.r10_slot);
    const int lhlo = A.center - R10_LH / 2, wlo = A.center - HWIN_REG / 2;
    for (int t = lane; t < R10_LHBYTES / 4; t += 32) lh[t] = 0;
    for (int t = threadIdx.x; t < HWIN_REG; t += blockDim.x) hwin[t] = 0;
    const R10Hist H = {(unsigned char*)(lh + lane), hwin, A.hist, lhlo, wlo};
    ws.init(lane);
    __syncthreads();

    const QuantParams Q = *A.qp;
    if (A.lor_fused) {
        // Lorenzo blocks first (k_quant_lor's work, a ticket per block): their long wavefront
        // chains overlap the regression blocks of the other warps.  Tile 0 holds the block,
        // tile 1 + the row table its float64 reconstruction, the bins go straight to global.
        const u32 nl = A.counters[4];
        for (;;) {
            u32 t = 0;
            if (lane == 0) t = atomicAdd(&A.counters[8], 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= nl) break;
            const long long bl = A.lor_list[t];
            lor_block<HWIN_REG>(A, Q, bl, A.dup_eval != 0, (float*)slot, (double*)(slot + S.tile_bytes),
                                A.bins + bins_index(g, bl, 0), hwin, wlo, lane);
            __syncwarp();
        }
        // generic-proxy writes to the tiles before the TMA (async proxy) writes them
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
    }
    // list positions: warp w of CTA c starts at c * nw + w, then takes tickets NW, NW + 1, ...
    // from counters[7] (dynamic: SMs that run ahead take more blocks).  The ticket is drawn two
    // blocks ahead by lane 4, the list entry it names arrives one block ahead; the next block's
    // tile is in flight while this one is processed.
    const u32 NW = gridDim.x * nw, nlist = A.counters[5];
    const u32 idx = blockIdx.x * nw + warp;
    u32 ticket = 0;
    auto draw = [&] {
        if (lane == 4) ticket = NW + atomicAdd(&A.counters[7], 1u);
    };
    // per-block global operands (coefficients twice: the duplicate's independent copy, the
    // checksum pair, the list entry after the next) travel one block ahead by cp.async into
    // the slot's two R10Pre records, so their latency hides behind a block's work
    auto prefetch = [&](long long bb, int q) {
        R10Pre* P = pre + q;
        if (lane == 0) cp_async16(&P->cf, A.coef + bb);
        else if (lane == 1 && DUP) cp_async16(&P->cg, A.coef + bb);
        else if (lane == 2 && PIN) cp_async8(&P->ins, A.insum + bb);
        else if (lane == 3 && PIN) cp_async8(&P->inis, A.inisum + bb);
        else if (lane == 4) {
            if (ticket < nlist) cp_async4(&P->nxt, A.r10_list + ticket);
            else P->nxt = ~0u;
        }
        cp_commit();
    };
    long long b = idx < nlist ? (long long)A.r10_list[idx] : -1ll;
    if (b >= 0) {
        draw();
        prefetch(b, 0);
        draw();
        ws.issue(A.x, g, S, &tmap, block_info(g, b), 0, lane);
    }
    u32 lh_load = 0;
    int buf = 0;
    while (b >= 0) {
        const BlockInfo B = block_info(g, b);
        cp_async_wait();
        __syncwarp();
        const R10Pre* P = pre + buf;
        const long long bnx = P->nxt == ~0u ? -1ll : (long long)P->nxt;
        const float4 cf = P->cf;
        const float4 cg = DUP ? P->cg : cf;   // the duplicate's independently loaded copy
        if (bnx >= 0) {
            prefetch(bnx, buf ^ 1);
            draw();
            ws.issue(A.x, g, S, &tmap, block_info(g, bnx), buf ^ 1, lane);
        }
        ws.wait(S, buf, bnx >= 0);
        float* tile = (float*)(slot + buf * S.tile_bytes);
        const int by = B.by, rows = B.bx * by, vol = B.vol, zoff = zshift(g, B), npairs = rows * 5;
        TileWalk w0;
        w0.bx = B.bx; w0.by = by; w0.bz = 10; w0.stride = S.tz; w0.zoff = zoff; w0.bye = S.tye;
        // working-array faults persist only without input protection (pipeline.py:331-361)
        if (!PIN && A.n_faults) apply_input_faults(A, b, tile, w0, lane);
        const double b3 = (double)cf.w;
        const double b3d = (double)cg.w;   // the duplicate's own copy of b3
        const float b3r = __double2float_rn(__dmul_rn(b3, (double)Q.rcp32));
        u16* gbins = A.bins + bins_index(g, b, 0);
        const bool hasdup = block_has_dup(A, b);
        bool mism = false, skip = false;
        R10Acc acc;
        // the lane's column of point pairs: z offsets k0, k0 + 1 of rows rsub, rsub + 6, ... (lanes
        // 30, 31 idle; 92% of the lane slots busy on a 10^3 block)
        r10_rowtab<DUP>(rowtab, rows, by, S.tye, S.tz, zoff, cf, cg, b3r, (double)Q.rcp32, lane);
        const int rsub = lane < 30 ? lane / 5 : R10_ROWS, k0 = 2 * (lane - 5 * (lane / 5));
        const float kf0 = (float)k0, kf1 = (float)(k0 + 1);
        const double ck0 = __dmul_rn(b3, int_to_f64(k0)), ck1 = __dmul_rn(b3, int_to_f64(k0 + 1));
        const double ckd0 = DUP ? __dmul_rn(b3d, int_to_f64(k0)) : ck0, ckd1 = DUP ? __dmul_rn(b3d, int_to_f64(k0 + 1)) : ck1;
        auto lane_points = [&](auto f) {
            for (int r = rsub; r < rows; r += 6) {
                f(10 * r + k0);
                f(10 * r + k0 + 1);
            }
        };
        const u32 cbin = (u32)Q.center - 0x4B400000u;   // bits(m) + cbin = center + RN(s)
        const u32 sink0 = H.sink();
        for (int pass = 0; pass < 2; pass++) {
            acc.reset();
            for (int r = rsub; r < rows; r += 6) {
                const R10Row R = rowtab[r];
                const float2 x2 = *(const float2*)(tile + R.toff + k0);   // 8-byte aligned (zoff 0 or 2)
                u32 r0, r1;
                const u32 b0 = r10_point<DUP>(Q, x2.x, kf0, ck0, ckd0, R, b3r, cbin, H, acc, r0);
                const u32 b1 = r10_point<DUP>(Q, x2.y, kf1, ck1, ckd1, R, b3r, cbin, H, acc, r1);
                const u32 p0 = (u32)(10 * r + k0);
                *(u32*)(gbins + p0) = __byte_perm(b0, b1, 0x5410);
                acc.bs += b0 + b1;
                acc.bis += p0 * b0 + (p0 + 1u) * b1;
                acc.dc += (u64)r0 + (u64)r1;
                if (PIN) {
                    const u32 u0 = __float_as_uint(x2.x), u1 = __float_as_uint(x2.y);
                    acc.cs += (u64)u0 + (u64)u1;
                    acc.csi += (u64)p0 * u0 + (u64)(p0 + 1u) * u1;
                }
            }
            // out-of-window fast bins of this lane (counted in its sink): recount into the CTA / global
            // window before the fix-up moves counts between bins
            if (__any_sync(0xffffffffu, H.sink() != sink0)) {
                if (H.sink() != sink0) {
                    H.set_sink(sink0);
                    // the lane's (<= 17) bin pairs, 9 loads in flight at a time
                    for (int h = 0; h < R10_ROWS / 6 + 1; h += 9) {
                        u32 wv[9];
#pragma unroll
                        for (int t = 0; t < 9; t++) {
                            const int r = rsub + 6 * (h + t);
                            wv[t] = r < rows ? *(const u32*)(gbins + 10 * r + k0) : (u32)H.lhlo * 0x10001u;
                        }
#pragma unroll
                        for (int t = 0; t < 9; t++) {
#pragma unroll
                            for (int u = 0; u < 2; u++) {
                                const u32 bb = (wv[t] >> (16 * u)) & 0xffffu;
                                if (bb - (u32)H.lhlo >= (u32)R10_LH) reg_hist_out(H.hwin, H.ghist, H.wlo, (int)bb, 1);
                            }
                        }
                    }
                }
                __syncwarp();
            }
            // exact recomputation of the flagged points (fix-up re-tests each point of the lane)
            const bool fl = acc.emax >= 0.49999905f || acc.amin <= Q.band32 || acc.macc != 0u || hasdup || !Q.fast32;
            if (__any_sync(0xffffffffu, fl)) {
                __syncwarp();
                if (fl) {
                    for (int r = rsub; r < rows; r += 6) {
                        const R10Row R = rowtab[r];
                        const double di = int_to_f64(R.ij >> 16), dj = int_to_f64(R.ij & 0xffff);
                        for (int u = 0; u < 2; u++) {
                            const int k = k0 + u;
                            r10_fix_point<DUP>(A, b, hasdup, Q, tile[R.toff + k], 10 * r + k, k, R.ab, R.ab2, R.abr,
                                               R.erow, b3r, di, dj, cf, cg, gbins, H, acc, mism);
                        }
                    }
                }
                __syncwarp();
            }
            if (!PIN || pass == 1) break;
            // stage (c) verification of the tile against the stage (a) pair (pipeline.py:331-361)
            const u64 cs = warp_sum_u64_redux(acc.cs), csi = warp_sum_u64_redux(acc.csi);
            if (cs == P->ins && csi == P->inis) break;
            // undo this pass's histogram counts, correct the tile, run again
            __syncwarp();
            lane_points([&](int p) { H.add(gbins[p], -1); });
            const int rr = tile_correct(tile, w0, vol, P->ins, P->inis, lane);
            if (lane == 0) {
                atomicAdd(&A.counters[3], 1u);
                A.events[b] |= rr == 1 ? 1 : 4;
            }
            if (rr != 1) {
                skip = true;
                break;
            }
            mism = false;
        }
        lh_load += 40u;   // per-lane counter increments of this block (<= 34)
        if (!skip) {
            const u32 bs = __reduce_add_sync(0xffffffffu, acc.bs);
            const u64 bis = warp_sum_u64_redux((u64)acc.bis), dc = warp_sum_u64_redux(acc.dc);
            if (__ballot_sync(0xffffffffu, mism) && lane == 0) atomicOr(&A.counters[1], 1u << (B.xid * 2 + 1));
            __syncwarp();
            // unpredictable words in point order (rare): 32 consecutive points per step
            u32 nz = 0;
            if (__any_sync(0xffffffffu, acc.nz)) {
                u32* unp = A.unp_scratch + (size_t)b * g.vmax;
                for (int p0 = 0; p0 < vol; p0 += 32) {
                    const int p = p0 + lane;
                    const bool z = p < vol && gbins[p] == 0u;
                    const unsigned m = __ballot_sync(0xffffffffu, z);
                    if (z) {
                        const int rr = p / 10, k = p - rr * 10, i = rr / by, j = rr - i * by;
                        unp[nz + __popc(m & ((1u << lane) - 1u))] = __float_as_uint(tile[(i * S.tye + j) * S.tz + zoff + k]);
                    }
                    nz += __popc(m);
                }
            }
            if (lane == 0) {
                A.unpc[b] = nz;
                if (nz) atomicAdd((u64*)&A.layout[LAYOUT_NUNP], (u64)nz);
                A.bsum[b] = bs;
                A.bisum[b] = bis;
                A.dcs[b] = dc;
            }
        }
        if (lh_load > 255u - 2u * 40u) {
            lh_flush10(lh, A.hist, lhlo, A.cap, lane);
            lh_load = 0;
        }
        buf ^= 1;
        b = bnx;
    }
    lh_flush10(lh, A.hist, lhlo, A.cap, lane);
    __syncthreads();
    for (int t = threadIdx.x; t < HWIN_REG; t += blockDim.x) {
        const u32 v = hwin[t];
        const int sy = wlo + t;
        if (v && sy >= 0 && sy < A.cap) atomicAdd(&A.hist[sy], (u64)v);
    }
}

}  // namespace ftlz
