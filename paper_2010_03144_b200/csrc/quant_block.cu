// quant_block.cu -- stage (c) of pipeline.compress for regression blocks (pipeline.py:390-409,
// 442-453): verify input, predict (duplicated), quantize, reconstruct (duplicated),
// double-check, bins / unpredictable words / checksums / sum_dc / histogram.
//
// Warp-autonomous: every warp owns a stream of blocks (static stride over the grid's warps),
// stages each block in shared memory with ONE TMA tensor copy (tma.cuh), double-buffered on
// an mbarrier, and processes it without any CTA-wide barrier.  Lane l takes the contiguous
// point range [l*c, l*c + c) of the block (c odd, so the 32 lanes' tile reads fall in distinct
// banks); the row prediction ((b0 + b1 i) + b2 j) comes from a per-block table and the k term
// b3*k from a second one, so the per-point work is the reference's float64 sequence plus an
// incremental walk.  The quantizer is branch-free (reciprocal multiply, 2^52-magic floor) and
// raises a flag within a few ulps of any decision threshold or on a duplicated-evaluation
// mismatch; such a point is recomputed with the exact reference formulation (blocks.cu
// quant_point), so the fast path never changes a result.  The stage (a) input checksum is
// accumulated in the same loop and verified afterwards; a mismatching block is corrected
// (checksum.py:109-142) and recomputed.  Histogram: lane-private 16-bit counters for the 64
// bins around the centre (conflict-free, no atomics), a CTA window, then global atomics.
namespace ftlz {

// quantize() contract (common.cuh) without branches; `slow` is raised instead of resolving
// an ambiguous point.  floor(fl(h + 0.5)) = RN(t) - (t < RN(t)) with RN(t) from t + 2^52
// and the exact residual d = t - RN(t); |d| < 2^-30 means t sits at an integer, where the
// reciprocal's <= 3 ulp error could change the floor.
FTLZ_DEV int quant_fast(double h_rcp, double diff, const QuantParams& Q, bool& ok, u32& slow) {
    double h = __dmul_rn(fabs(diff), h_rcp);
    u64 hb = dbits(h);
    bool small = hb <= Q.capd2_bits;
    slow |= ((u32)(hb >> 32) - (u32)(Q.capd2_bits >> 32) + 1u) < 2u;  // h' within 2^-20 rel of 2*cap
    double t = __dadd_rn(h, 0.5);
    double m = __dadd_rn(t, 4503599627370496.0);   // 2^52: low word = RN(t)
    double r = __dadd_rn(m, -4503599627370496.0);
    double d = __dadd_rn(t, -r);                   // exact (Sterbenz)
    u32 dhi = (u32)(dbits(d) >> 32);
    int q = (int)(u32)dbits(m) - (int)(dhi >> 31);
    slow |= (u32)(small && ((dhi & 0x7fffffffu) < 0x3e100000u));
    q = small ? q : 0;
    int s = (int)(u32)(dbits(diff) >> 32) >> 31;   // 0 or -1
    q = (q ^ s) - s;
    int b = Q.center + q;
    ok = small && (u32)(b - 1) < (u32)(Q.cap - 1);
    return ok ? b : 0;
}

FTLZ_DEV float4 ld_volatile_f4(const float4* p) {
    float4 v;
    asm volatile("ld.volatile.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

// ---- lane-private histogram window around the centre: counter of bin o for lane l at
//      lh16[o * 32 + l] (lanes never share a counter; no atomics).  LH8: 128 bins of u8
//      counters (flushed every few blocks), else 64 bins of u16 counters.
#ifndef LH16
#define LH8
#endif
#ifdef LH8
#ifndef LH8_BINS
#define LH8_BINS 128
#endif
#define LH_BINS LH8_BINS
typedef unsigned char LHT;
#define LH_MAXC 255u
#else
#define LH_BINS 64
typedef u16 LHT;
#define LH_MAXC 65535u
#endif
#define HWIN_REG 2048

FTLZ_DEV void reg_hist_out(u32* hwin, u64* ghist, int wlo, int bin, int delta) {
    unsigned ow = (unsigned)(bin - wlo);
    if (ow < HWIN_REG) atomicAdd(&hwin[ow], (u32)delta);
    else atomicAdd(&ghist[bin], (u64)(long long)delta);
}
FTLZ_DEV void reg_hist_add(LHT* lh16, u32* hwin, u64* ghist, int lhlo, int wlo, int bin, int lane, int delta) {
    unsigned o = (unsigned)(bin - lhlo);
    if (o < LH_BINS) lh16[o * 32 + lane] += (LHT)delta;
    else reg_hist_out(hwin, ghist, wlo, bin, delta);
}

#ifdef LH8
// lane l sums bins lhlo + 4l .. + 3 over the 32 lane counters (8 words of 4 bytes each) and
// clears them
FTLZ_DEV void reg_hist_flush_lanes(LHT* lh16, u64* ghist, int lhlo, int cap, int lane) {
    __syncwarp();
    u32* w32 = (u32*)lh16;   // bin o occupies words o*8 .. o*8+7
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int o = 4 * lane + q;
        if (o >= LH_BINS) break;
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
#else
// lane l sums bins lhlo + 2l and lhlo + 2l + 1 over the 32 lane counters and clears them
FTLZ_DEV void reg_hist_flush_lanes(LHT* lh16, u64* ghist, int lhlo, int cap, int lane) {
    __syncwarp();
    u32* w32 = (u32*)lh16;   // bin o occupies words o*16 .. o*16+15
    u32 lo = 0, hi = 0;
#pragma unroll 4
    for (int q = 0; q < 16; q++) {
        int c = (q + lane) & 15;
        u32 a = w32[(2 * lane) * 16 + c], b = w32[(2 * lane + 1) * 16 + c];
        w32[(2 * lane) * 16 + c] = 0;
        w32[(2 * lane + 1) * 16 + c] = 0;
        lo += (a & 0xffffu) + (a >> 16);
        hi += (b & 0xffffu) + (b >> 16);
    }
    int b0 = lhlo + 2 * lane;
    if (lo && b0 >= 0 && b0 < cap) atomicAdd(&ghist[b0], (u64)lo);
    if (hi && b0 + 1 >= 0 && b0 + 1 < cap) atomicAdd(&ghist[b0 + 1], (u64)hi);
    __syncwarp();
}
#endif

// per-lane partial sums of one block
struct RegAcc {
    u64 cs, csi, bis, dc;
    u32 bs, nz;
    u32 flagged;   // some point of this lane needs the exact formulation
    u32 outwin;    // some bin of this lane lies outside the lane-private window
};

// lane-private counter of an in-window bin; out-of-window bins go to the sink row LH_BINS
FTLZ_DEV void lh_bump(LHT* lh16, int lhlo, int bin, int lane, u32& outwin) {
    unsigned o = (unsigned)(bin - lhlo);
    const bool in = o < LH_BINS;
    outwin |= (u32)!in;
    o = in ? o : LH_BINS;
    lh16[o * 32 + lane] += 1;
}

// position of a point inside the block / tile
struct RegPos {
    int i, j, k, rp, t;
};

struct RegBlk {
    const float* tile;
    const double *abt, *abt2, *ctab, *ctab2;
    u16* bins16;
    int by, bz, tjump, ijump;
};

// fast path for one point: bin, reconstructed value, ambiguity flag
template <bool DUP>
FTLZ_DEV u32 reg_point_fast(const QuantParams& Q, float x32, double ab, double ab2, double ck, double ck2, float& r32,
                            u32& slow) {
    const double x64 = (double)x32;
    const double p1 = __dadd_rn(ab, ck);
    bool ok;
    slow = (u32)Q.exact_div;
    int bin = quant_fast(Q.rcp, __dadd_rn(x64, -p1), Q, ok, slow);
    const double offs = int_to_f64(ok ? bin - Q.center : -Q.center);
    const double d1 = __dadd_rn(p1, __dmul_rn(Q.twoeb, offs));
    if (DUP) {
        // second evaluation from independently loaded operands (ab2, twoeb_dup)
        const double p2 = __dadd_rn(ab2, ck2);
        const double d2 = __dadd_rn(p2, __dmul_rn(Q.twoeb_dup, offs));
        const u64 xx = (dbits(p1) ^ dbits(p2)) | (dbits(d1) ^ dbits(d2));
        slow |= (u32)xx | (u32)(xx >> 32);
    }
    const float d32 = __double2float_rn(d1);
    const bool keep = ok && fabs(__dadd_rn(x64, -(double)d32)) <= Q.eb;
    r32 = keep ? d32 : x32;
    return keep ? (u32)bin : 0u;
}

// one step of the point walk (branch-free): k, then the row (j), then i
template <bool FULLJ>
FTLZ_DEV void reg_step(RegPos& P, const RegBlk& K) {
    P.k++;
    P.t++;
    const bool w = P.k == K.bz;
    P.k = w ? 0 : P.k;
    P.t += w ? K.tjump : 0;
    P.rp += (int)w;
    if (!FULLJ) {
        P.j += (int)w;
        const bool w2 = P.j == K.by;
        P.j = w2 ? 0 : P.j;
        P.t += w2 ? K.ijump : 0;
    }
}

// points [p0, pend) starting at position P; accumulates into acc.  FULLJ: the block spans the
// tile's whole j extent (no i-step jump), true for all but the last block row of a ragged field.
// Points go in groups of RB: all RB points' operands are loaded before any store of the group,
// so the RB float64 dependency chains interleave (the bins / histogram stores would otherwise
// order every point after the previous one's stores).
#ifndef RB
#define RB 4
#endif
template <bool DUP, bool PIN, bool FULLJ>
FTLZ_DEV void reg_points(const QuantParams& Q, const RegBlk& K, RegPos P, int p0, int pend, int lane, LHT* lh16,
                         u32* hwin, u64* ghist, int lhlo, int wlo, RegAcc& acc) {
    u32 flag = 0, outw = 0;
    int p = p0;
    for (; p + RB <= pend; p += RB) {
        float x[RB];
        double ab[RB], ab2[RB], ck[RB], ck2[RB];
#pragma unroll
        for (int u = 0; u < RB; u++) {
            x[u] = K.tile[P.t];
            ab[u] = K.abt[P.rp];
            ab2[u] = DUP ? K.abt2[P.rp] : ab[u];
            ck[u] = K.ctab[P.k];
            ck2[u] = DUP ? K.ctab2[P.k] : ck[u];
            reg_step<FULLJ>(P, K);
        }
        u32 fb[RB];
        float r32[RB];
#pragma unroll
        for (int u = 0; u < RB; u++) {
            u32 slow;
            fb[u] = reg_point_fast<DUP>(Q, x[u], ab[u], ab2[u], ck[u], ck2[u], r32[u], slow);
            flag |= slow;
        }
#pragma unroll
        for (int u = 0; u < RB; u++) {
            const u32 pu = (u32)(p + u);
            if (PIN) {
                const u32 xu = __float_as_uint(x[u]);
                acc.cs += (u64)xu;
                acc.csi += (u64)pu * (u64)xu;
            }
            K.bins16[p + u] = (u16)fb[u];
            acc.bs += fb[u];
            acc.bis += (u64)pu * (u64)fb[u];
            acc.dc += (u64)__float_as_uint(r32[u]);
            acc.nz += fb[u] == 0u;
            lh_bump(lh16, lhlo, (int)fb[u], lane, outw);
        }
    }
    for (; p < pend; p++) {
        const float x32 = K.tile[P.t];
        const double ab = K.abt[P.rp], ab2 = DUP ? K.abt2[P.rp] : ab;
        if (PIN) {
            const u32 u = __float_as_uint(x32);
            acc.cs += (u64)u;
            acc.csi += (u64)(u32)p * (u64)u;
        }
        float r32;
        u32 slow;
        const u32 fb = reg_point_fast<DUP>(Q, x32, ab, ab2, K.ctab[P.k], DUP ? K.ctab2[P.k] : K.ctab[P.k], r32, slow);
        flag |= slow;
        K.bins16[p] = (u16)fb;
        acc.bs += fb;
        acc.bis += (u64)(u32)p * (u64)fb;
        acc.dc += (u64)__float_as_uint(r32);
        acc.nz += fb == 0u;
        lh_bump(lh16, lhlo, (int)fb, lane, outw);
        reg_step<FULLJ>(P, K);
    }
    acc.flagged = flag;
    acc.outwin = outw;
}

// out-of-window bins of this lane's range (after any fixup): CTA window / global atomics
FTLZ_DEV void reg_hist_outwin(const u16* bins16, int p0, int pend, u32* hwin, u64* ghist, int lhlo, int wlo) {
    for (int p = p0; p < pend; p++) {
        const int bin = bins16[p];
        if ((unsigned)(bin - lhlo) >= LH_BINS) reg_hist_out(hwin, ghist, wlo, bin, 1);
    }
}

// exact recomputation of the ambiguous points of this lane (rare): rescan the range with the
// fast path and replace every flagged point's results by the exact formulation's; points with
// injected duplicated-evaluation faults (hasdup) always take the exact formulation
template <bool DUP>
FTLZ_DEV void reg_fixup(const CompArgs& A, long long b, bool hasdup, const QuantParams& Q, const RegBlk& K,
                        const float4& cf, int p0, int pend, int zoff, int tz, int tye, int lane, LHT* lh16, u32* hwin,
                        u64* ghist, int lhlo, int wlo, RegAcc& acc, bool& mism) {
    for (int p = p0; p < pend; p++) {
        const int rp = p / K.bz, k = p - rp * K.bz, i = rp / K.by, j = rp - i * K.by;
        const float x32 = K.tile[(i * tye + j) * tz + zoff + k];
        const double ab = K.abt[rp], ab2 = DUP ? K.abt2[rp] : ab, ck = K.ctab[k], ck2 = DUP ? K.ctab2[k] : ck;
        float rf;
        u32 slow;
        const u32 fb_fast = reg_point_fast<DUP>(Q, x32, ab, ab2, ck, ck2, rf, slow);
        DupMask M;
        const bool fp = hasdup && dup_masks(A, b, p, M);
        if (!slow && !fp) continue;
        if (!fp) {
#pragma unroll
            for (int r = 0; r < 3; r++) M.p[r] = M.r[r] = 0ull;
        }
        float rx;
        double back;
        // evaluation 1 from the row / k tables, 2 from their independently built copies, 3 from
        // the float32 coefficients (pipeline.py:392-394 re-evaluates _regression_grid_batch)
        const u32 fb = (u32)quant_point(
            Q, x32, __dadd_rn(ab, ck), DUP, [&] { return __dadd_rn(opaque(ab2), opaque(ck2)); },
            [&] {
                return __dadd_rn(__dadd_rn(__dadd_rn((double)cf.x, __dmul_rn((double)cf.y, int_to_f64(i))),
                                           __dmul_rn((double)cf.z, int_to_f64(j))),
                                 __dmul_rn(opaque((double)cf.w), int_to_f64(k)));
            },
            M, &rx, &mism, &back);
        K.bins16[p] = (u16)fb;
        acc.bs += fb - fb_fast;
        acc.bis += (u64)(u32)p * (u64)fb - (u64)(u32)p * (u64)fb_fast;
        acc.dc += (u64)__float_as_uint(rx) - (u64)__float_as_uint(rf);
        acc.nz += (u32)(fb == 0u) - (u32)(fb_fast == 0u);
        // lane window: drop the fast bin, count the exact one (out-of-window: post pass)
        unsigned of = (unsigned)((int)fb_fast - lhlo), ox = (unsigned)((int)fb - lhlo);
        if (of < LH_BINS) lh16[of * 32 + lane] -= 1;
        else lh16[LH_BINS * 32 + lane] -= 1;
        if (ox < LH_BINS) lh16[ox * 32 + lane] += 1;
        else acc.outwin = 1;
    }
}

#ifndef QR_WARPS
#define QR_WARPS 12
#endif
__global__ void __launch_bounds__(QR_WARPS * 32, 1) k_quant_reg(const __grid_constant__ CompArgs A,
                                                       const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // 128-byte aligned base for the TMA destinations
    unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const Geom& g = A.g;
    if (dev_failed(A.st)) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const StageCfg S = A.stage;
    unsigned char* slot = smem + (size_t)warp * A.qr_slot;
    WarpStager ws;
    ws.base = slot;
    ws.tbytes = S.tile_bytes;
    u16* bins16 = (u16*)(slot + 2 * S.tile_bytes);
    double* abt = (double*)(slot + A.qr_tab);
    double* abt2 = abt + A.rmax;
    double* ctab = abt2 + A.rmax;
    double* ctab2 = ctab + 64;
    LHT* lh16 = (LHT*)(ctab2 + 64);
    ws.bar = (u64*)(lh16 + (LH_BINS + 1) * 32);
    u32* hwin = (u32*)(smem + (size_t)nw * A.qr_slot);
    const int wlo = A.center - HWIN_REG / 2, lhlo = A.center - LH_BINS / 2;
    for (int t = threadIdx.x; t < HWIN_REG; t += blockDim.x) hwin[t] = 0;
    for (int t = lane; t < (LH_BINS + 1) * 32 * (int)sizeof(LHT) / 4; t += 32) ((u32*)lh16)[t] = 0;
    ws.init(lane);
    __syncthreads();

    const QuantParams Q = *A.qp;
    const bool dup = A.dup_eval != 0, pin = A.protect_input != 0;
    const long long NW = (long long)gridDim.x * nw;
    // the regression blocks k_quant_reg10 does not take (regx_list, built by k_reglist)
    const u32 nlist = A.counters[6];
    u32 idx = blockIdx.x * nw + warp;
    auto next_reg = [&](long long) {
        const long long r = idx < nlist ? (long long)A.regx_list[idx] : (long long)g.nb;
        idx += (u32)NW;
        return r;
    };
    u32 lh_load = 0;   // max per-lane count added since the last flush
    long long b = next_reg(0);
    BlockInfo Bnext = block_info(g, b);
    if (b < g.nb) ws.issue(A.x, g, S, &tmap, Bnext, 0, lane);
    int buf = 0;
    while (b < g.nb) {
        const BlockInfo B = Bnext;
        const long long bn = next_reg(b + NW);
        if (bn < g.nb) {
            Bnext = block_info(g, bn);
            ws.issue(A.x, g, S, &tmap, Bnext, buf ^ 1, lane);
        }
        ws.wait(S, buf, bn < g.nb);
        float* tile = (float*)(slot + buf * S.tile_bytes);
        const int bx = B.bx, by = B.by, bz = B.bz, vol = B.vol, rows = bx * by;
        TileWalk w0;
        w0.bx = bx; w0.by = by; w0.bz = bz; w0.stride = S.tz; w0.zoff = zshift(g, B); w0.bye = S.tye;
        // working-array faults persist only without input protection (pipeline.py:331-361)
        if (!pin && A.n_faults) apply_input_faults(A, b, tile, w0, lane);
        // per-block tables: row term ((b0 + b1 i) + b2 j), twice from independent loads; b3*k
        const float4 cf = A.coef[b];
        const float4 cg = dup ? ld_volatile_f4(A.coef + b) : cf;
        const FastDiv& fby = by == g.e ? A.fd_e : A.fd_ry;
        const FastDiv& fbz = bz == g.e ? A.fd_e : A.fd_rz;
        for (int r = lane; r < rows; r += 32) {
            int i = (int)fdiv((u32)r, fby), j = r - i * by;
            double di = int_to_f64(i), dj = int_to_f64(j);
            abt[r] = __dadd_rn(__dadd_rn((double)cf.x, __dmul_rn((double)cf.y, di)), __dmul_rn((double)cf.z, dj));
            if (dup)
                abt2[r] = __dadd_rn(__dadd_rn((double)cg.x, __dmul_rn((double)cg.y, di)), __dmul_rn((double)cg.z, dj));
        }
        for (int k = lane; k < bz; k += 32) {
            ctab[k] = __dmul_rn((double)cf.w, int_to_f64(k));
            if (dup) ctab2[k] = __dmul_rn((double)cg.w, int_to_f64(k));
        }
        __syncwarp();

        const int chunk = ((vol + 31) >> 5) | 1;
        const int p0 = lane * chunk, pend = min(p0 + chunk, vol);
        RegPos P0 = {0, 0, 0, 0, 0};
        if (p0 < vol) {
            P0.rp = (int)fdiv((u32)p0, fbz);
            P0.k = p0 - P0.rp * bz;
            P0.i = (int)fdiv((u32)P0.rp, fby);
            P0.j = P0.rp - P0.i * by;
        }
        P0.t = (P0.i * S.tye + P0.j) * S.tz + w0.zoff + P0.k;
        RegBlk K;
        K.tile = tile; K.abt = abt; K.abt2 = abt2; K.ctab = ctab; K.ctab2 = ctab2; K.bins16 = bins16;
        const bool hasdup = block_has_dup(A, b);
        K.by = by; K.bz = bz; K.tjump = S.tz - bz; K.ijump = (S.tye - by) * S.tz;
        RegAcc acc;
        bool mism = false, skip = false;
        for (int pass = 0; pass < 2; pass++) {
            acc.cs = acc.csi = acc.bis = acc.dc = 0;
            acc.bs = acc.nz = 0;
            const bool fullj = by == S.tye;
            if (dup) {
                if (pin) {
                    if (fullj) reg_points<true, true, true>(Q, K, P0, p0, pend, lane, lh16, hwin, A.hist, lhlo, wlo, acc);
                    else reg_points<true, true, false>(Q, K, P0, p0, pend, lane, lh16, hwin, A.hist, lhlo, wlo, acc);
                } else {
                    reg_points<true, false, false>(Q, K, P0, p0, pend, lane, lh16, hwin, A.hist, lhlo, wlo, acc);
                }
            } else {
                if (pin) reg_points<false, true, false>(Q, K, P0, p0, pend, lane, lh16, hwin, A.hist, lhlo, wlo, acc);
                else reg_points<false, false, false>(Q, K, P0, p0, pend, lane, lh16, hwin, A.hist, lhlo, wlo, acc);
            }
            if (hasdup) acc.flagged = 1;
            if (__any_sync(0xffffffffu, acc.flagged != 0)) {
                if (acc.flagged) {
                    if (dup) reg_fixup<true>(A, b, hasdup, Q, K, cf, p0, pend, w0.zoff, S.tz, S.tye, lane, lh16, hwin, A.hist, lhlo, wlo, acc, mism);
                    else reg_fixup<false>(A, b, hasdup, Q, K, cf, p0, pend, w0.zoff, S.tz, S.tye, lane, lh16, hwin, A.hist, lhlo, wlo, acc, mism);
                }
            }
            if (__any_sync(0xffffffffu, acc.outwin != 0) && acc.outwin)
                reg_hist_outwin(bins16, p0, pend, hwin, A.hist, lhlo, wlo);
            if (!pin || pass == 1) break;
            // stage (c) verification of the re-read input against the stage (a) pair
            const u64 cs = warp_sum_u64(acc.cs), csi = warp_sum_u64(acc.csi);
            if (cs == A.insum[b] && csi == A.inisum[b]) break;
            for (int p = p0; p < pend; p++) reg_hist_add(lh16, hwin, A.hist, lhlo, wlo, bins16[p], lane, -1);
            int rr = tile_correct(tile, w0, vol, A.insum[b], A.inisum[b], lane);
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
        lh_load += (u32)chunk;
        if (!skip) {
            const u32 nz = acc.nz;
            const u32 nzt = warp_sum_u32(nz);
            const u32 bs = warp_sum_u32(acc.bs);
            const u64 bis = warp_sum_u64(acc.bis);
            const u64 dc = warp_sum_u64(acc.dc);
            if (__ballot_sync(0xffffffffu, mism) && lane == 0) atomicOr(&A.counters[1], 1u << (B.xid * 2 + 1));
            if (lane == 0) {
                A.unpc[b] = nzt;
                if (nzt) atomicAdd((u64*)&A.layout[LAYOUT_NUNP], (u64)nzt);
                A.bsum[b] = bs;
                A.bisum[b] = bis;
                A.dcs[b] = dc;
            }
            __syncwarp();
            // bins to the encoder layout, 16 bytes per lane-step
            const int nch = (vol + 7) >> 3;
            for (int c = lane; c < nch; c += 32)
                *(uint4*)(A.bins + bins_index(g, b, 8 * c)) = *(const uint4*)(bins16 + 8 * c);
            if (nzt) {
                // unpredictable words in point order: lanes own contiguous ranges
                u32 pre = nz;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    u32 v = __shfl_up_sync(0xffffffffu, pre, o);
                    if (lane >= o) pre += v;
                }
                pre -= nz;
                u32* unp = A.unp_scratch + (size_t)b * g.vmax;
                RegPos P = P0;
                for (int p = p0; p < pend && nz; p++) {
                    if (bins16[p] == 0) unp[pre++] = __float_as_uint(tile[P.t]);
                    P.k++;
                    P.t++;
                    if (P.k == bz) {
                        P.k = 0;
                        P.j++;
                        P.t += K.tjump;
                        if (P.j == by) {
                            P.j = 0;
                            P.t += K.ijump;
                        }
                    }
                }
            }
        }
        if (lh_load > LH_MAXC - 2u * ((((u32)g.vmax + 31u) >> 5) | 1u)) {
            reg_hist_flush_lanes(lh16, A.hist, lhlo, A.cap, lane);
            lh_load = 0;
        }
        buf ^= 1;
        b = bn;
    }
    reg_hist_flush_lanes(lh16, A.hist, lhlo, A.cap, lane);
    __syncthreads();
    for (int t = threadIdx.x; t < HWIN_REG; t += blockDim.x) {
        u32 v = hwin[t];
        int s = wlo + t;
        if (v && s >= 0 && s < A.cap) atomicAdd(&A.hist[s], (u64)v);
    }
}

}  // namespace ftlz
