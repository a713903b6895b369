// quant_reg10.cu -- stage (c) of pipeline.compress for regression blocks whose z rows hold 10
// points (the default block edge; pipeline.py:390-453, quantize.py:37-52, duplicated
// evaluation pipeline.py:157-179), one lane per (i, j) row.
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
// two TMA tiles (tma.cuh); lane l takes rows l, l + 32, ... of the block.  A row's ten floats
// arrive in three vector loads (12-float tile rows: conflict-free), its bins leave as five
// 32-bit stores straight into the encoder's bins array.  Histogram: lane-private u8 counters
// for the 64 bins around the centre (flushed every few blocks), out-of-window bins counted by
// a rescan of the lane's rows.
namespace ftlz {

#ifndef R10_WARPS
#define R10_WARPS 12
#endif
#define R10_LH 256   // lane-private histogram window (bins center - 128 .. center + 127) + a sink row

struct R10Acc {
    u32 bs;        // sum of bins
    u64 bis;       // sum of p * bin
    u64 dc;        // sum of recon32 words
    u64 cs, csi;   // input checksum pair
    u32 rowflag;   // bit t: row lane + 32 t has a flagged point
    u32 rownz;     // bit t: row lane + 32 t has an unpredictable point
};

// lane-private u8 counters: bin o of the window at byte o * 32 + lane.  A bin outside the window
// only bumps the lane's sink counter (row R10_LH): no branch in the point loop; a row whose
// sink count moved is recounted afterwards into the CTA's shared window (hwin, HWIN_REG bins) or,
// beyond it, the global histogram.
struct R10Hist {
    unsigned char* lhw;   // this lane's column of the u8 window
    u32* hwin;            // CTA window
    u64* ghist;
    int lhlo, wlo;
    // count `delta` (+1 / -1) for bin b (slow paths: fix-up, tail, undo)
    FTLZ_DEV void add(u32 b, int delta) const {
        const u32 o = b - (u32)lhlo;
        if (o < (u32)R10_LH) lhw[o * 32] += (unsigned char)delta;
        else reg_hist_out(hwin, ghist, wlo, (int)b, delta);
    }
    // hot path: window counter, or the sink for an out-of-window bin (recounted per row)
    FTLZ_DEV void bump(u32 b) const { lhw[min(b - (u32)lhlo, (u32)R10_LH) * 32] += 1; }
    FTLZ_DEV u32 sink() const { return lhw[R10_LH * 32]; }
};

FTLZ_DEV void lh_flush10(unsigned char* lh, u64* ghist, int lhlo, int cap, int lane) {
    __syncwarp();
    u32* w32 = (u32*)lh;   // bin o: words o * 8 .. o * 8 + 7 (32 u8 counters)
#pragma unroll
    for (int q = 0; q < R10_LH / 32; q++) {
        const int o = (R10_LH / 32) * lane + q;
        u32 sum = 0;
#pragma unroll
        for (int c = 0; c < 8; c++) {
            const int cc = (c + lane) & 7;
            sum = __dp4a(w32[o * 8 + cc], 0x01010101u, sum);
            w32[o * 8 + cc] = 0;
        }
        const int bn = lhlo + o;
        if (sum && bn >= 0 && bn < cap) atomicAdd(&ghist[bn], (u64)sum);
    }
    __syncwarp();
}

// one point of the fast path (see the file header); accumulates into the row sums
template <bool DUP, bool PIN>
FTLZ_DEV u32 r10_point(const QuantParams& Q, float x, int k, float kf, double kd, double ab, double ab2, double b3,
                       double b3d, float b3r, float abr, float erow, u32 cbin, const R10Hist& H, float& emax,
                       float& amin, u32& macc, bool& nzf, u32& bsr, u32& kbr, u32& rbits, u64& kxr) {
    // float32 estimate of S and its distance to the nearest half-integer
    const float c = __fmaf_rn(b3r, kf, abr);
    const float s = __fmaf_rn(x, Q.rcp32, -c);
    const float m = __fadd_rn(s, 12582912.0f);   // 1.5 * 2^23: low mantissa bits = RN(s)
    const float f = __fadd_rn(s, -__fadd_rn(m, -12582912.0f));
    const bool big = !(fabsf(s) < Q.sbig);
    emax = fmaxf(emax, big ? 0.0f : __fadd_rn(fabsf(f), __fmaf_rn(fabsf(s), 4.76837158203125e-07f, erow)));
    const u32 bin = __float_as_uint(m) + cbin;
    const bool ok = !big && (bin - 1u) < (u32)(Q.cap - 1);
    // float64 reconstruction in the reference order
    const double offs = __int2double_rn((int)(bin - (u32)Q.center));
    const double p1 = __dadd_rn(ab, __dmul_rn(b3, kd));
    const double d1 = __dadd_rn(p1, __dmul_rn(Q.twoeb, offs));
    if (DUP) {
        const double p2 = __dadd_rn(ab2, __dmul_rn(b3d, kd));
        const double d2 = __dadd_rn(p2, __dmul_rn(Q.twoeb_dup, offs));
        const u64 xp = dbits(p1) ^ dbits(p2), xd = dbits(d1) ^ dbits(d2);
        macc |= (u32)xp | (u32)(xp >> 32) | (u32)xd | (u32)(xd >> 32);
    }
    const float d32 = __double2float_rn(d1);
    const float a = __fadd_rn(fabsf(__fadd_rn(x, -d32)), -Q.eb32);
    amin = fminf(amin, ok ? fabsf(a) : INFINITY);
    const bool keep = ok && a <= 0.0f;
    const u32 b = keep ? bin : 0u;
    const float r32 = keep ? d32 : x;
    nzf |= !keep;
    bsr += b;
    kbr += (u32)k * b;
    rbits = __float_as_uint(r32);
    if (PIN) kxr += (u64)(u32)k * (u64)__float_as_uint(x);
    H.bump(b);
    return b;
}

// one row (i, j) of a regression block: 10 points as 5 pairs (two points in flight keep the
// register footprint small enough for more resident warps); returns the row's flag bits
// (bit 0: some point needs the exact formulation, bit 1: some point is unpredictable)
template <bool DUP, bool PIN>
FTLZ_DEV u32 r10_row(const QuantParams& Q, const float* row, double ab, double ab2, double b3, double b3d,
                     float b3r, int p0, u16* gbins, const R10Hist& H, R10Acc& acc) {
    const float abr = __double2float_rn(__dmul_rn(ab, (double)Q.rcp32));
    const float erow = __fmaf_rn(9.0f, fabsf(b3r), fabsf(abr)) * 9.5367431640625e-07f + 9.094947017729282e-13f;
    const u32 cbin = (u32)Q.center - 0x4B400000u;   // bits(m) + cbin = center + RN(s)
    float emax = 0.0f, amin = INFINITY;
    u32 macc = 0, bsr = 0, kbr = 0;
    bool nzf = false;
    u64 dcr = 0, csr = 0, kxr = 0;
    u32* gw = (u32*)(gbins + p0);   // p0 = 10 r: 4-byte aligned
    const u32 sink0 = H.sink();
    float kf = 0.0f;
    double kd = 0.0;
#pragma unroll 1
    for (int k = 0; k < 10; k += 2) {
        const float2 x2 = *(const float2*)(row + k);   // row start is 8-byte aligned (zoff 0 or 2)
        u32 r0, r1;
        const u32 b0 = r10_point<DUP, PIN>(Q, x2.x, k, kf, kd, ab, ab2, b3, b3d, b3r, abr, erow, cbin, H, emax,
                                           amin, macc, nzf, bsr, kbr, r0, kxr);
        const u32 b1 = r10_point<DUP, PIN>(Q, x2.y, k + 1, __fadd_rn(kf, 1.0f), __dadd_rn(kd, 1.0), ab, ab2, b3, b3d,
                                           b3r, abr, erow, cbin, H, emax, amin, macc, nzf, bsr, kbr, r1, kxr);
        gw[k >> 1] = b0 | (b1 << 16);
        // 64-bit sums of word pairs: one three-input add with carries per pair
        dcr += (u64)r0 + (u64)r1;
        if (PIN) csr += (u64)__float_as_uint(x2.x) + (u64)__float_as_uint(x2.y);
        kf = __fadd_rn(kf, 2.0f);
        kd = __dadd_rn(kd, 2.0);
    }
    acc.bs += bsr;
    acc.bis += (u64)(u32)p0 * (u64)bsr + (u64)kbr;
    acc.dc += dcr;
    if (PIN) {
        acc.cs += csr;
        acc.csi += (u64)(u32)p0 * csr + kxr;
    }
    if (H.sink() != sink0) {
        // out-of-window bins of this row: move them from the sink to the CTA / global counts
        H.lhw[R10_LH * 32] = (unsigned char)sink0;
        for (int k = 0; k < 10; k++) {
            const u32 bb = gbins[p0 + k];
            if (bb - (u32)H.lhlo >= (u32)R10_LH) reg_hist_out(H.hwin, H.ghist, H.wlo, (int)bb, 1);
        }
    }
    const bool fl = emax >= 0.49999905f || amin <= Q.band32 || macc != 0u;
    return (fl ? 1u : 0u) | (nzf ? 2u : 0u);
}

// exact recomputation of the flagged rows of this lane (reference formulation, blocks.cu
// quant_point): replaces the fast results of every point whose fast evaluation was flagged,
// or that carries an injected duplicated-evaluation fault
template <bool DUP>
FTLZ_DEV void r10_fixup(const CompArgs& A, long long b, bool hasdup, const QuantParams& Q, const float* tile, int tye,
                        int tz, int zoff, int rows, const FastDiv& fby, int by, const float4& cf, const float4& cg,
                        u16* gbins, const R10Hist& H, int lane, R10Acc& acc, bool& mism) {
    const float b3r = __double2float_rn(__dmul_rn((double)cf.w, (double)Q.rcp32));
    for (int t = 0, r = lane; r < rows; t++, r += 32) {
        if (!((acc.rowflag >> t) & 1u)) continue;
        const int i = (int)fdiv((u32)r, fby), j = r - i * by;
        const float* row = tile + (i * tye + j) * tz + zoff;
        const double di = int_to_f64(i), dj = int_to_f64(j);
        const double ab = __dadd_rn(__dadd_rn((double)cf.x, __dmul_rn((double)cf.y, di)), __dmul_rn((double)cf.z, dj));
        const double ab2 = DUP ? __dadd_rn(__dadd_rn((double)cg.x, __dmul_rn((double)cg.y, di)), __dmul_rn((double)cg.z, dj)) : ab;
        const float abr = __double2float_rn(__dmul_rn(ab, (double)Q.rcp32));
        const float erow = __fmaf_rn(9.0f, fabsf(b3r), fabsf(abr)) * 9.5367431640625e-07f + 9.094947017729282e-13f;
        for (int k = 0; k < 10; k++) {
            const int p = r * 10 + k;
            const float x = row[k];
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
            if (!(edge || unsure || mis || fp)) continue;
            if (!fp) {
#pragma unroll
                for (int q = 0; q < 3; q++) M.p[q] = M.r[q] = 0ull;
            }
            float rx;
            double back;
            const u32 ex = (u32)quant_point(
                Q, x, p1, DUP, [&] { return __dadd_rn(opaque(ab2), opaque(ck2k)); },
                [&] {
                    return __dadd_rn(__dadd_rn(__dadd_rn((double)cf.x, __dmul_rn((double)cf.y, di)),
                                               __dmul_rn((double)cf.z, dj)),
                                     __dmul_rn(opaque((double)cf.w), int_to_f64(k)));
                },
                M, &rx, &mism, &back);
            gbins[p] = (u16)ex;
            acc.bs += ex - fb;
            acc.bis += (u64)(u32)p * (u64)ex - (u64)(u32)p * (u64)fb;
            acc.dc += (u64)__float_as_uint(rx) - (u64)__float_as_uint(rf);
            if (ex == 0u) acc.rownz |= 1u << t;
            // drop the fast bin's count, count the exact bin
            H.add(fb, -1);
            H.add(ex, 1);
        }
    }
}

// tail points (rows past the last full 32-row iteration, at most 12 rows): one point per lane
// per step, by the reference formulation directly (blocks.cu quant_point; no fix-up needed)
template <bool DUP, bool PIN>
FTLZ_DEV void r10_tail_point(const CompArgs& A, long long b, bool hasdup, const QuantParams& Q, const float* tile,
                             int tye, int tz, int zoff, int p, int by, const float4& cf, const float4& cg,
                             u16* gbins, const R10Hist& H, R10Acc& acc, bool& mism) {
    const int rr = p / 10, k = p - rr * 10, i = rr / by, j = rr - i * by;
    const float x = tile[(i * tye + j) * tz + zoff + k];
    const double di = int_to_f64(i), dj = int_to_f64(j), dk = int_to_f64(k);
    auto pred = [&](const float4& c) {
        return __dadd_rn(__dadd_rn(__dadd_rn((double)c.x, __dmul_rn((double)c.y, di)), __dmul_rn((double)c.z, dj)),
                         __dmul_rn((double)c.w, dk));
    };
    DupMask M;
    if (!(hasdup && dup_masks(A, b, p, M))) {
#pragma unroll
        for (int q = 0; q < 3; q++) M.p[q] = M.r[q] = 0ull;
    }
    float r32;
    double back;
    const u32 bin = (u32)quant_point(
        Q, x, pred(cf), DUP, [&] { return pred(cg); },
        [&] {
            return __dadd_rn(__dadd_rn(__dadd_rn((double)cf.x, __dmul_rn((double)cf.y, di)), __dmul_rn((double)cf.z, dj)),
                             __dmul_rn(opaque((double)cf.w), dk));
        },
        M, &r32, &mism, &back);
    gbins[p] = (u16)bin;
    acc.bs += bin;
    acc.bis += (u64)(u32)p * (u64)bin;
    acc.dc += (u64)__float_as_uint(r32);
    if (bin == 0u) acc.rownz = 1u;
    if (PIN) {
        const u32 u = __float_as_uint(x);
        acc.cs += (u64)u;
        acc.csi += (u64)(u32)p * (u64)u;
    }
    H.add(bin, 1);
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
    unsigned char* lh = slot + 2 * S.tile_bytes;   // (R10_LH + 1) x 32 u8 counters
    ws.bar = (u64*)(lh + (R10_LH + 1) * 32);
    u32* hwin = (u32*)(smem + (size_t)nw * A.r10_slot);
    const int lhlo = A.center - R10_LH / 2, wlo = A.center - HWIN_REG / 2;
    for (int t = lane; t < (R10_LH + 1) * 8; t += 32) ((u32*)lh)[t] = 0;
    for (int t = threadIdx.x; t < HWIN_REG; t += blockDim.x) hwin[t] = 0;
    const R10Hist H = {lh + lane, hwin, A.hist, lhlo, wlo};
    ws.init(lane);
    __syncthreads();

    const QuantParams Q = *A.qp;
    // blocks idx, idx + NW, ... of r10_list (k_reglist); the next block's tile is in flight
    // while this one is processed
    const u32 NW = gridDim.x * nw, nlist = A.counters[5];
    u32 idx = blockIdx.x * nw + warp;
    auto list_at = [&](u32 i) { return i < nlist ? (long long)A.r10_list[i] : (long long)-1; };
    long long b = list_at(idx);
    if (b >= 0) ws.issue(A.x, g, S, &tmap, block_info(g, b), 0, lane);
    u32 lh_load = 0;
    int buf = 0;
    while (b >= 0) {
        const BlockInfo B = block_info(g, b);
        idx += NW;
        const long long bnx = list_at(idx);
        if (bnx >= 0) ws.issue(A.x, g, S, &tmap, block_info(g, bnx), buf ^ 1, lane);
        ws.wait(S, buf, bnx >= 0);
        const float4 cf = A.coef[b];
        float* tile = (float*)(slot + buf * S.tile_bytes);
        const int by = B.by, rows = B.bx * by, vol = B.vol, zoff = zshift(g, B);
        // rows in 32-row steps, lane = row; a short remainder (<= 12 rows) point by point
#ifdef R10_TAIL
        const int nfull = (rows & 31) <= 12 ? (rows & ~31) : rows;
#else
        const int nfull = rows;
#endif
        TileWalk w0;
        w0.bx = B.bx; w0.by = by; w0.bz = 10; w0.stride = S.tz; w0.zoff = zoff; w0.bye = S.tye;
        // working-array faults persist only without input protection (pipeline.py:331-361)
        if (!PIN && A.n_faults) apply_input_faults(A, b, tile, w0, lane);
        const float4 cg = DUP ? ld_volatile_f4(A.coef + b) : cf;
        const double b0 = (double)cf.x, b1 = (double)cf.y, b2 = (double)cf.z, b3 = (double)cf.w;
        const double b3d = (double)cg.w;   // the duplicate's own copy of b3
        const float b3r = __double2float_rn(__dmul_rn(b3, (double)Q.rcp32));
        const FastDiv& fby = by == g.e ? A.fd_e : A.fd_ry;
        u16* gbins = A.bins + bins_index(g, b, 0);
        const bool hasdup = block_has_dup(A, b);
        bool mism = false, skip = false;
        R10Acc acc;
        // every point this lane owns: its rows (< nfull), then its tail points
        auto lane_points = [&](auto f) {
            for (int r = lane; r < nfull; r += 32)
                for (int k = 0; k < 10; k++) f(r * 10 + k);
            for (int p = nfull * 10 + lane; p < vol; p += 32) f(p);
        };
        for (int pass = 0; pass < 2; pass++) {
            acc.bs = 0; acc.bis = 0; acc.dc = 0; acc.cs = 0; acc.csi = 0;
            acc.rowflag = 0; acc.rownz = 0;
            for (int t = 0, r = lane; r < nfull; t++, r += 32) {
                const int i = (int)fdiv((u32)r, fby), j = r - i * by;
                const double di = __int2double_rn(i), dj = __int2double_rn(j);
                const double ab = __dadd_rn(__dadd_rn(b0, __dmul_rn(b1, di)), __dmul_rn(b2, dj));
                const double ab2 = DUP ? __dadd_rn(__dadd_rn((double)cg.x, __dmul_rn((double)cg.y, di)),
                                                   __dmul_rn((double)cg.z, dj))
                                       : ab;
                const float* row = tile + (i * S.tye + j) * S.tz + zoff;
                const u32 rf = r10_row<DUP, PIN>(Q, row, ab, ab2, b3, b3d, b3r, r * 10, gbins, H, acc);
                acc.rowflag |= (rf & 1u) << t;
                acc.rownz |= rf >> 1;
            }
            for (int p = nfull * 10 + lane; p < vol; p += 32)
                r10_tail_point<DUP, PIN>(A, b, hasdup, Q, tile, S.tye, S.tz, zoff, p, by, cf, cg, gbins, H, acc, mism);
            if (hasdup) acc.rowflag = ~0u;
            if (!Q.fast32) acc.rowflag = ~0u;
            if (__any_sync(0xffffffffu, acc.rowflag != 0)) {
                __syncwarp();
                if (acc.rowflag)
                    r10_fixup<DUP>(A, b, hasdup, Q, tile, S.tye, S.tz, zoff, nfull, fby, by, cf, cg, gbins, H,
                                   lane, acc, mism);
                __syncwarp();
            }
            if (!PIN || pass == 1) break;
            // stage (c) verification of the tile against the stage (a) pair (pipeline.py:331-361)
            const u64 cs = warp_sum_u64_redux(acc.cs), csi = warp_sum_u64_redux(acc.csi);
            if (cs == A.insum[b] && csi == A.inisum[b]) break;
            // undo this pass's histogram counts, correct the tile, run again
            __syncwarp();
            lane_points([&](int p) { H.add(gbins[p], -1); });
            const int rr = tile_correct(tile, w0, vol, A.insum[b], A.inisum[b], lane);
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
        lh_load += 4u * 10u;   // per-lane counter increments of this block (<= 40)
        if (!skip) {
            const u32 bs = __reduce_add_sync(0xffffffffu, acc.bs);
            const u64 bis = warp_sum_u64_redux(acc.bis), dc = warp_sum_u64_redux(acc.dc);
            if (__ballot_sync(0xffffffffu, mism) && lane == 0) atomicOr(&A.counters[1], 1u << (B.xid * 2 + 1));
            __syncwarp();
            // unpredictable words in point order (rare): 32 consecutive points per step
            u32 nz = 0;
            if (__any_sync(0xffffffffu, acc.rownz != 0)) {
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
