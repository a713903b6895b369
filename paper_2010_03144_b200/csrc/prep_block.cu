// prep_block.cu -- stage (a) + (b) of pipeline.compress (pipeline.py:295-373): value range
// (core.py:72-74), input checksums (checksum.py:171-181), regression fit with numpy's pairwise
// float64 summation (predict.py:81-104), sampled predictor selection (predict.py:196-231).
//
// Warp-autonomous like k_quant_reg: every warp streams its blocks through two TMA-staged tiles
// (tma.cuh) and reduces each block without CTA barriers.  The four fit sums follow numpy's
// pairwise order exactly: lanes own the 8-way unrolled chains of the host-built leaves
// (Leaf: start, len, ncomb), chains are combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by
// shuffles, tails are added in order, and the leaf tree is folded by a post-order program --
// one lane per sum, stack in shared memory.  Each element is visited exactly once, so the
// checksum pair and the value range ride along.
namespace ftlz {

// post-order fold of per-leaf partial sums: lane v < NV folds column v (stack in shared memory)
template <int NV>
FTLZ_DEV void fold_leaves(const Leaf* leaves, int nleaf, const double* leafval, double* stk, double out[NV],
                          int lane) {
    double mine = 0.0;
    if (lane < NV) {
        int sp = 0;
        for (int l = 0; l < nleaf; l++) {
            double v = leafval[l * NV + lane];
            int nc = __ldg(&leaves[l].ncomb);
            for (int t = 0; t < nc; t++) {
                sp--;
                v = __dadd_rn(stk[sp * NV + lane], v);
            }
            stk[sp * NV + lane] = v;
            sp++;
        }
        mine = __dadd_rn(0.0, stk[lane]);
    }
#pragma unroll
    for (int v = 0; v < NV; v++) out[v] = __shfl_sync(0xffffffffu, mine, v);
}

// (i, j, k, t) walker over a block held in a TMA tile, stepping `step` points in p order
struct PWalk {
    int i, j, k, t;
    // from the plan's coordinate table entry i | j << 8 | k << 16
    FTLZ_DEV void set_crd(u32 c, int tye, int tz, int zoff) {
        i = (int)(c & 0xffu);
        j = (int)((c >> 8) & 0xffu);
        k = (int)(c >> 16);
        t = (i * tye + j) * tz + zoff + k;
    }
    FTLZ_DEV void set(int p, int by, int bz, int tye, int tz, int zoff) {
        int rp = p / bz;
        k = p - rp * bz;
        i = rp / by;
        j = rp - i * by;
        t = (i * tye + j) * tz + zoff + k;
    }
    // d <= bz: at most one row carry (branch-free)
    FTLZ_DEV void step1(int d, int by, int bz, int tjump, int ijump) {
        k += d;
        t += d;
        const bool w = k >= bz;
        k -= w ? bz : 0;
        t += w ? tjump : 0;
        j += (int)w;
        const bool w2 = j == by;
        j = w2 ? 0 : j;
        i += (int)w2;
        t += w2 ? ijump : 0;
    }
    FTLZ_DEV void step(int d, int by, int bz, int tjump, int ijump) {
        k += d;
        t += d;
        while (k >= bz) {
            k -= bz;
            j++;
            t += tjump;
            if (j == by) {
                j = 0;
                i++;
                t += ijump;
            }
        }
    }
};

struct PrepAcc {
    u64 cs, csi;
    float mx, mn;
    u32 nan;
};

FTLZ_DEV void prep_visit(const float* tile, const PWalk& w, int p, const double* cv, int cvn, PrepAcc& a, double t4[4]) {
    const float f = tile[w.t];
    const u32 u = __float_as_uint(f);
    a.cs += (u64)u;
    a.csi += (u64)(u32)p * (u64)u;
    a.nan |= (u32)(f != f);
    a.mx = fmaxf(a.mx, f);
    a.mn = fminf(a.mn, f);
    const double v = (double)f;
    t4[0] = v;
    t4[1] = __dmul_rn(cv[w.i], v);
    t4[2] = __dmul_rn(cv[cvn + w.j], v);
    t4[3] = __dmul_rn(cv[2 * cvn + w.k], v);
}

// ---- exact-sum path of the fit ------------------------------------------------------------
// numpy's pairwise order (predict.py:81-104) only matters when some partial sum rounds.  Every
// summand c * v (c = idx - (n - 1) / 2, v = float64(x)) is a multiple of G / 2, G = the ulp of
// the block's smallest nonzero |x|, and every partial sum of any order is bounded by
// 2 (e - 1) vol max|x|.  When that bound is below 2^52 G (ExtPlan::exl, tested per block on the
// exponents of max |x| and min nonzero |x|), every partial sum -- numpy's and ours -- is exact,
// so the four sums can be formed in any order.  Here: lane = row (i, j); per row R = sum_k v,
// T = sum_k sum_{k' < k} v_k' (so sum_k (k - hz) v = hz R - T), then S(ci v) = sum (i - hx) R,
// S(cj v) = sum (j - hy) R, S(ck v) = sum (hz R - T); any failing block takes the pairwise path.

FTLZ_DEV void madw(u64& acc, u32 a, u32 b) {   // acc += a * b (one IMAD.WIDE.U32)
    asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}

struct ExactAcc {
    double R, T;
    u64 W, K;
    u32 amax, amin;
};

FTLZ_DEV void exact_point(float x, u32 k, ExactAcc& e, PrepAcc& acc) {
    const u32 u = __float_as_uint(x);
    madw(e.W, u, 1u);
    madw(e.K, u, k);
    acc.mx = fmaxf(acc.mx, x);
    acc.mn = fminf(acc.mn, x);
    const u32 a = u & 0x7fffffffu;
    e.amax = max(e.amax, a);
    e.amin = min(e.amin, a - 1u);   // zero -> 0xffffffff: ignored
    e.T = __dadd_rn(e.T, e.R);
    e.R = __dadd_rn(e.R, (double)x);
}

// one 10-float row of a TMA tile whose rows start at z shift ZO (0 or 2): three vector loads
// (16-byte rows groups of 12-float tile rows fall in distinct bank quads: conflict-free)
template <int ZO>
FTLZ_DEV void load_row10(const float* row, float v[10]) {
    if (ZO == 0) {
        const float4 a = *(const float4*)row, b = *(const float4*)(row + 4);
        const float2 c = *(const float2*)(row + 8);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
        v[8] = c.x; v[9] = c.y;
    } else {
        const float2 a = *(const float2*)row;
        const float4 b = *(const float4*)(row + 2), c = *(const float4*)(row + 6);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = b.z; v[5] = b.w; v[6] = c.x; v[7] = c.y;
        v[8] = c.z; v[9] = c.w;
    }
}

// rows of the block: ZO = 0 / 2 for 10-float rows, -1 generic
template <int ZO>
FTLZ_DEV void exact_rows(const float* tile, int rows, int by, int bz, int tye, int tz, int zoff, const FastDiv& fby,
                         double hx, double hy, double hz, int lane, PrepAcc& acc, double s4[4], u64& cs, u64& csi,
                         u32& amax, u32& amin) {
    ExactAcc e;
    e.amax = 0u;
    e.amin = 0xffffffffu;
    for (int r = lane; r < rows; r += 32) {
        const int i = (int)fdiv((u32)r, fby), j = r - i * by;
        const float* row = tile + (i * tye + j) * tz + zoff;
        e.R = 0.0;
        e.T = 0.0;
        e.W = 0ull;
        e.K = 0ull;
        if (ZO >= 0) {
            float v[10];
            load_row10<ZO>(row, v);
#pragma unroll
            for (int k = 0; k < 10; k++) exact_point(v[k], (u32)k, e, acc);
        } else {
            for (int k = 0; k < bz; k++) exact_point(row[k], (u32)k, e, acc);
        }
        s4[0] = __dadd_rn(s4[0], e.R);
        s4[1] = __dadd_rn(s4[1], __dmul_rn(__dadd_rn(int_to_f64(i), -hx), e.R));
        s4[2] = __dadd_rn(s4[2], __dmul_rn(__dadd_rn(int_to_f64(j), -hy), e.R));
        s4[3] = __dadd_rn(s4[3], __dadd_rn(__dmul_rn(hz, e.R), -e.T));
        cs += e.W;
        csi += (u64)(u32)(r * bz) * e.W + e.K;
    }
    amax = e.amax;
    amin = e.amin;
}

// returns true (warp-uniform) when the exact path applies; then sums, cs, csi are final
FTLZ_DEV bool prep_exact(const float* tile, const ExtPlan& PL, int by, int bz, int tye, int tz, int zoff,
                         const FastDiv& fby, int lane, PrepAcc& acc, double sums[4], u64& cs, u64& csi) {
    const int rows = PL.bx * by;
    const double hx = 0.5 * (double)(PL.bx - 1), hy = 0.5 * (double)(by - 1), hz = 0.5 * (double)(bz - 1);
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    u64 c0 = 0, c1 = 0;
    u32 amax, amin;
    if (bz == 10 && (tz & 3) == 0 && zoff == 0)
        exact_rows<0>(tile, rows, by, bz, tye, tz, zoff, fby, hx, hy, hz, lane, acc, s4, c0, c1, amax, amin);
    else if (bz == 10 && (tz & 3) == 0 && zoff == 2)
        exact_rows<2>(tile, rows, by, bz, tye, tz, zoff, fby, hx, hy, hz, lane, acc, s4, c0, c1, amax, amin);
    else
        exact_rows<-1>(tile, rows, by, bz, tye, tz, zoff, fby, hx, hy, hz, lane, acc, s4, c0, c1, amax, amin);
    amax = __reduce_max_sync(0xffffffffu, amax);
    amin = __reduce_min_sync(0xffffffffu, amin);
    acc.nan |= (u32)(amax > 0x7f800000u);
    cs = warp_sum_u64_redux(c0);
    csi = warp_sum_u64_redux(c1);
    if (amax >= 0x7f800000u) return false;   // inf / NaN: the pairwise path
    if (amin != 0xffffffffu) {
        const int emax = (int)(amax >> 23), emin = max((int)((amin + 1u) >> 23), 1);
        if (emax - emin + PL.exl > 28) return false;
    }
    // butterfly: lane bits 4, 3 select which of the four sums a lane keeps (exact: any order)
    const bool h4 = lane & 16, h3 = lane & 8;
    double k0 = h4 ? s4[2] : s4[0], k1 = h4 ? s4[3] : s4[1];
    k0 = __dadd_rn(k0, __shfl_xor_sync(0xffffffffu, h4 ? s4[0] : s4[2], 16));
    k1 = __dadd_rn(k1, __shfl_xor_sync(0xffffffffu, h4 ? s4[1] : s4[3], 16));
    double v = __dadd_rn(h3 ? k1 : k0, __shfl_xor_sync(0xffffffffu, h3 ? k0 : k1, 8));
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    v = __dadd_rn(0.0, v);   // exact; +0.0 for a zero sum, as numpy's 0.0 + S
    // sum q lives in lanes 8 q .. 8 q + 7 (q = 2 bit4 + bit3)
#pragma unroll
    for (int q = 0; q < 4; q++) sums[q] = __shfl_sync(0xffffffffu, v, 8 * q);
    return true;
}

// one tile per warp: the next block's TMA is issued as soon as the current tile is last read,
// and the freed shared memory buys more resident warps (latency hiding across warps)
#define PREP_NBUF 1
#define PREP_STK 16   // post-order fold depth: log2(leaves) + 1 <= 13 for 64^3 blocks

__global__ void __launch_bounds__(640, 1) k_prep(const __grid_constant__ CompArgs A, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const Geom& g = A.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const StageCfg S = A.stage;
    unsigned char* slot = smem + (size_t)warp * A.pp_slot;
    WarpStager ws;
    ws.base = slot;
    ws.tbytes = S.tile_bytes;
    const int cvn = g.e;
    double* cv = (double*)(slot + PREP_NBUF * S.tile_bytes);   // [0,e) i - hx, [e,2e) j - hy, [2e,3e) k - hz
    double* stk = cv + 3 * cvn;                        // fold stack: depth <= PREP_STK, x 4
    double* leafval = stk + 4 * PREP_STK;              // nls x 4
    double* ar = leafval + 4 * A.pp_nls;               // samples
    double* al = ar + A.pp_ns;
    double* ptab = al + A.pp_ns;                       // b1 i, b2 j, b3 k (3 e entries)
    ws.bar = (u64*)(ptab + 3 * cvn);
    __shared__ u32 omx, omn, cta_nan, cta_nreg;
    if (threadIdx.x == 0) { omx = 0; omn = 0xffffffffu; cta_nan = 0; cta_nreg = 0; }
    ws.init(lane);
    __syncthreads();

    PrepAcc acc;
    acc.mx = -INFINITY;
    acc.mn = INFINITY;
    acc.nan = 0;
    u32 nreg = 0;
    int last_xid = -1;
    const long long NW = (long long)gridDim.x * nw;
    // blocks [pb0, pb1): the whole field, or one slab of block layers whose input has arrived
    const long long pb1 = A.pb1;
    long long b = A.pb0 + (long long)blockIdx.x * nw + warp;
    BlockInfo Bnext = block_info(g, b);
    if (b < pb1) ws.issue(A.x, g, S, &tmap, Bnext, 0, lane);
    int buf = 0;
    while (b < pb1) {
        const BlockInfo B = Bnext;
        const long long bn = b + NW;
        if (PREP_NBUF == 2 && bn < pb1) {
            Bnext = block_info(g, bn);
            ws.issue(A.x, g, S, &tmap, Bnext, buf ^ 1, lane);
        }
        ws.wait(S, buf, PREP_NBUF == 2 && bn < pb1);
        bool issued = false;
        float* tile = (float*)(slot + buf * S.tile_bytes);
        const int bx = B.bx, by = B.by, bz = B.bz, vol = B.vol;
        const int zoff = zshift(g, B), tjump = S.tz - bz, ijump = (S.tye - by) * S.tz;
        const ExtPlan& PL = A.plans[B.xid];
        const u32* crd = A.coords + PL.coord_off;
        if (B.xid != last_xid) {
            // centred coordinates c = idx - (n - 1) / 2 (predict.py:90-98)
            const double hx = (double)(bx - 1) / 2.0, hy = (double)(by - 1) / 2.0, hz = (double)(bz - 1) / 2.0;
            for (int t = lane; t < cvn; t += 32) {
                cv[t] = __dadd_rn(int_to_f64(t), -hx);
                cv[cvn + t] = __dadd_rn(int_to_f64(t), -hy);
                cv[2 * cvn + t] = __dadd_rn(int_to_f64(t), -hz);
            }
            last_xid = B.xid;
            __syncwarp();
        }
        // ---- one pass over every element: pairwise chains of S(v), S(ci v), S(cj v), S(ck v),
        //      input checksum pair and value range
        acc.cs = 0;
        acc.csi = 0;
        double sums[4];
        u64 cs, csi;
        const FastDiv& fby = by == g.e ? A.fd_e : A.fd_ry;
        const bool exact = prep_exact(tile, PL, by, bz, S.tye, S.tz, zoff, fby, lane, acc, sums, cs, csi);
        if (exact) {
            // exact sums, checksum pair and range from the row pass
        } else if (vol < 8) {
            double r[4] = {0.0, 0.0, 0.0, 0.0};
            if (lane == 0) {
                PWalk w;
                w.set(0, by, bz, S.tye, S.tz, zoff);
                for (int p = 0; p < vol; p++) {
                    double t4[4];
                    prep_visit(tile, w, p, cv, cvn, acc, t4);
#pragma unroll
                    for (int q = 0; q < 4; q++) r[q] = __dadd_rn(r[q], t4[q]);
                    w.step(1, by, bz, tjump, ijump);
                }
#pragma unroll
                for (int q = 0; q < 4; q++) r[q] = __dadd_rn(0.0, r[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; q++) sums[q] = __shfl_sync(0xffffffffu, r[q], 0);
        } else {
            const Leaf* leaves = A.leaves + PL.leaf_off;
            const int nchains = PL.nleaf * 8;
            for (int c0 = 0; c0 < nchains; c0 += 32) {
                const int c = c0 + lane;
                const int leaf = c >> 3, j8 = c & 7;
                double r[4] = {0.0, 0.0, 0.0, 0.0};
                int start = 0, len = 0;
                if (c < nchains) {
                    const Leaf Lf = leaves[leaf];
                    start = Lf.start;
                    len = Lf.len;
                    const int len8 = len - (len & 7);
                    PWalk w;
                    w.set_crd(__ldg(crd + start + j8), S.tye, S.tz, zoff);
                    prep_visit(tile, w, start + j8, cv, cvn, acc, r);
                    if (bz >= 8) {   // at most one row carry per step (the loop-invariant test hoisted)
#pragma unroll 2
                        for (int p = start + j8 + 8; p < start + len8; p += 8) {
                            w.step1(8, by, bz, tjump, ijump);
                            double t4[4];
                            prep_visit(tile, w, p, cv, cvn, acc, t4);
#pragma unroll
                            for (int q = 0; q < 4; q++) r[q] = __dadd_rn(r[q], t4[q]);
                        }
                    } else {
                        for (int p = start + j8 + 8; p < start + len8; p += 8) {
                            w.step(8, by, bz, tjump, ijump);
                            double t4[4];
                            prep_visit(tile, w, p, cv, cvn, acc, t4);
#pragma unroll
                            for (int q = 0; q < 4; q++) r[q] = __dadd_rn(r[q], t4[q]);
                        }
                    }
                }
                // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)): the lower lane is the left operand
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        double other = __shfl_xor_sync(0xffffffffu, r[q], o);
                        r[q] = (j8 & o) ? __dadd_rn(other, r[q]) : __dadd_rn(r[q], other);
                    }
                }
                if (j8 == 0 && c < nchains) {
                    const int len8 = len - (len & 7);
                    if (len8 < len) {
                        PWalk w;
                        w.set_crd(__ldg(crd + start + len8), S.tye, S.tz, zoff);
                        for (int p = start + len8; p < start + len; p++) {
                            double t4[4];
                            prep_visit(tile, w, p, cv, cvn, acc, t4);
#pragma unroll
                            for (int q = 0; q < 4; q++) r[q] = __dadd_rn(r[q], t4[q]);
                            w.step(1, by, bz, tjump, ijump);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; q++) leafval[leaf * 4 + q] = r[q];
                }
            }
            __syncwarp();
            fold_leaves<4>(leaves, PL.nleaf, leafval, stk, sums, lane);
        }
        if (!exact) {   // the pairwise path's visits recomputed the checksum pair
            cs = warp_sum_u64(acc.cs);
            csi = warp_sum_u64(acc.csi);
        }
        // ---- coefficients (batch form, predict.py:90-104): slopes on lanes 1..3, mean on lane 0
        float4 cf;
        {
            // lane 0: mean = S(v) / vol; lanes 1..3: slope = S(c v) / den, one division for all four
            double sl = 0.0, corr = 0.0, out0 = 0.0;
            const int ax = lane - 1;
            if (lane <= 3) {
                const double num = lane == 0 ? sums[0] : (lane == 1 ? sums[1] : (lane == 2 ? sums[2] : sums[3]));
                const double den = lane == 0 ? (double)vol : PL.den[ax];
                const double qd = __ddiv_rn(num, den);
                if (lane == 0) out0 = qd;
                else {
                    const int e = ax == 0 ? bx : (ax == 1 ? by : bz);
                    if (e != 1) {
                        sl = qd;
                        corr = __dmul_rn(__dmul_rn(sl, (double)(e - 1)), 0.5);   // x / 2.0 == x * 0.5 exactly
                    }
                }
            }
            const double s1 = __shfl_sync(0xffffffffu, sl, 1), s2 = __shfl_sync(0xffffffffu, sl, 2),
                         s3 = __shfl_sync(0xffffffffu, sl, 3);
            const double k1 = __shfl_sync(0xffffffffu, corr, 1), k2 = __shfl_sync(0xffffffffu, corr, 2),
                         k3 = __shfl_sync(0xffffffffu, corr, 3);
            out0 = __shfl_sync(0xffffffffu, out0, 0);
            // axes with extent 1 contribute nothing (predict.py: slope 0, no correction)
            if (bx != 1) out0 = __dadd_rn(out0, -k1);
            if (by != 1) out0 = __dadd_rn(out0, -k2);
            if (bz != 1) out0 = __dadd_rn(out0, -k3);
            cf = make_float4(__double2float_rn(out0), __double2float_rn(s1), __double2float_rn(s2), __double2float_rn(s3));
        }
        // ---- hooks after stage (a): COEFFS_FITTED, INPUT_AFTER_CHECKSUM (pipeline.py:328-329)
        TileWalk w0;
        w0.bx = bx; w0.by = by; w0.bz = bz; w0.stride = S.tz; w0.zoff = zoff; w0.bye = S.tye;
        bool bad = false;
        const long long bb = B.b;
        if (A.n_faults && A.fault_first[bb] >= 0) {
            const int f0 = A.fault_first[bb];
            for (int f = f0; f < A.n_faults && A.faults[f].block == bb; f++)
                if (A.faults[f].target == FTLZ_FAULT_COEFF) {
                    float* c4 = (float*)&cf;
                    c4[A.faults[f].element] = __uint_as_float(__float_as_uint(c4[A.faults[f].element]) ^ (1u << A.faults[f].bit));
                }
            if (apply_input_faults(A, bb, tile, w0, lane) && A.protect_input) {
                // stage (b) verification against the stage (a) checksum (pipeline.py:331-361)
                const int r = tile_correct(tile, w0, vol, cs, csi, lane);
                if (r == 1 && lane == 0) { A.events[bb] |= 1; atomicAdd(&A.counters[3], 1u); }
                if (r == 2) {
                    bad = true;
                    if (lane == 0) { A.events[bb] |= 4; atomicAdd(&A.counters[3], 1u); }
                }
            }
            __syncwarp();
        }
        if (!bad) {
            // ---- sampled selection (predict.py:196-231): samples at p = 8, 16, ...
            const int ns = PL.ns;
            const double c0 = (double)cf.x;
            // b1 i, b2 j, b3 k for the block's coordinates (predict.py:196-231 evaluates
            // ((b0 + b1 i) + b2 j) + b3 k with these same float64 products)
            for (int u = lane; u < 3 * cvn; u += 32) {
                const int ax = u / cvn, t = u - ax * cvn;
                const float cw = ax == 0 ? cf.y : (ax == 1 ? cf.z : cf.w);
                ptab[u] = __dmul_rn((double)cw, int_to_f64(t));
            }
            __syncwarp();
            const int sr = S.tz, sp = S.tye * S.tz;   // tile offsets of (j-1) and (i-1)
            for (int q = lane; q < ns; q += 32) {
                PWalk w;
                w.set_crd(__ldg(crd + 8 * (q + 1)), S.tye, S.tz, zoff);
                const int i = w.i, j = w.j, k = w.k, ad = w.t;
                const double v = (double)tile[ad];
                const double pr = __dadd_rn(__dadd_rn(__dadd_rn(c0, ptab[i]), ptab[cvn + j]), ptab[2 * cvn + k]);
                const double d100 = i > 0 ? (double)tile[ad - sp] : 0.0;
                const double d010 = j > 0 ? (double)tile[ad - sr] : 0.0;
                const double d001 = k > 0 ? (double)tile[ad - 1] : 0.0;
                const double d110 = (i > 0 && j > 0) ? (double)tile[ad - sp - sr] : 0.0;
                const double d101 = (i > 0 && k > 0) ? (double)tile[ad - sp - 1] : 0.0;
                const double d011 = (j > 0 && k > 0) ? (double)tile[ad - sr - 1] : 0.0;
                const double d111 = (i > 0 && j > 0 && k > 0) ? (double)tile[ad - sp - sr - 1] : 0.0;
                const double pl = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(d100, d010), d001), -d110), -d101), -d011), d111);
                ar[q] = fabs(__dadd_rn(v, -pr));
                al[q] = fabs(__dadd_rn(v, -pl));
            }
            __syncwarp();
            if (PREP_NBUF == 1 && bn < pb1) {   // the tile is free: start the next block's copy
                Bnext = block_info(g, bn);
                ws.issue(A.x, g, S, &tmap, Bnext, 0, lane);
                issued = true;
            }
            double e2[2];
            if (ns < 8) {
                double r0 = 0.0, r1 = 0.0;
                if (lane == 0) {
                    for (int q = 0; q < ns; q++) { r0 = __dadd_rn(r0, ar[q]); r1 = __dadd_rn(r1, al[q]); }
                    r0 = __dadd_rn(0.0, r0);
                    r1 = __dadd_rn(0.0, r1);
                }
                e2[0] = __shfl_sync(0xffffffffu, r0, 0);
                e2[1] = __shfl_sync(0xffffffffu, r1, 0);
            } else if (PL.nsleaf == 1) {
                // one pairwise leaf (ns <= 128): lanes 0-7 carry the eight chains of e_reg, lanes
                // 8-15 those of e_lor; ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7)) by
                // shuffles, the tail in order, then 0.0 + S
                const int j8 = lane & 7;
                const double* src = lane < 8 ? ar : al;
                const int len8 = ns - (ns & 7);
                double r = 0.0;
                if (lane < 16) {
                    r = src[j8];
                    for (int p = j8 + 8; p < len8; p += 8) r = __dadd_rn(r, src[p]);
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
                    const double other = __shfl_xor_sync(0xffffffffu, r, o);
                    r = (j8 & o) ? __dadd_rn(other, r) : __dadd_rn(r, other);
                }
                if (lane == 0 || lane == 8) {
                    for (int p = len8; p < ns; p++) r = __dadd_rn(r, src[p]);
                    r = __dadd_rn(0.0, r);
                }
                e2[0] = __shfl_sync(0xffffffffu, r, 0);
                e2[1] = __shfl_sync(0xffffffffu, r, 8);
            } else {
                const Leaf* sl = A.leaves + PL.sleaf_off;
                const int nchains = PL.nsleaf * 8;
                for (int c0c = 0; c0c < nchains; c0c += 32) {
                    const int c = c0c + lane;
                    const int leaf = c >> 3, j8 = c & 7;
                    double r[2] = {0.0, 0.0};
                    int start = 0, len = 0;
                    if (c < nchains) {
                        const Leaf Lf = sl[leaf];
                        start = Lf.start;
                        len = Lf.len;
                        const int len8 = len - (len & 7);
                        r[0] = ar[start + j8];
                        r[1] = al[start + j8];
                        for (int p = start + j8 + 8; p < start + len8; p += 8) {
                            r[0] = __dadd_rn(r[0], ar[p]);
                            r[1] = __dadd_rn(r[1], al[p]);
                        }
                    }
#pragma unroll
                    for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
                        for (int q = 0; q < 2; q++) {
                            double other = __shfl_xor_sync(0xffffffffu, r[q], o);
                            r[q] = (j8 & o) ? __dadd_rn(other, r[q]) : __dadd_rn(r[q], other);
                        }
                    }
                    if (j8 == 0 && c < nchains) {
                        const int len8 = len - (len & 7);
                        for (int p = start + len8; p < start + len; p++) {
                            r[0] = __dadd_rn(r[0], ar[p]);
                            r[1] = __dadd_rn(r[1], al[p]);
                        }
                        leafval[leaf * 2] = r[0];
                        leafval[leaf * 2 + 1] = r[1];
                    }
                }
                __syncwarp();
                fold_leaves<2>(sl, PL.nsleaf, leafval, stk, e2, lane);
            }
            double er = e2[0], el = e2[1];
            if (A.n_faults && A.fault_first[bb] >= 0) {
                const int f0 = A.fault_first[bb];
                for (int f = f0; f < A.n_faults && A.faults[f].block == bb; f++) {
                    if (A.faults[f].target != FTLZ_FAULT_ESTIMATE) continue;
                    const u64 bit = 1ull << A.faults[f].bit;
                    if (A.faults[f].element == 0) er = __longlong_as_double((long long)(dbits(er) ^ bit));
                    else el = __longlong_as_double((long long)(dbits(el) ^ bit));
                }
            }
            int kind = er < el ? 1 : 0;
            if (A.override_ && A.override_[bb] >= 0) kind = A.override_[bb];
            if (lane == 0) {
                A.coef[bb] = cf;
                A.insum[bb] = cs;
                A.inisum[bb] = csi;
                A.ind[bb] = (u8)kind;
                if (kind == 1) nreg++;
                else A.lor_list[atomicAdd(&A.counters[4], 1u)] = (u32)bb;
            }
        } else if (lane == 0) {
            A.ind[bb] = 0;
            A.coef[bb] = cf;
        }
        __syncwarp();
        if (PREP_NBUF == 1 && !issued && bn < pb1) {
            Bnext = block_info(g, bn);
            ws.issue(A.x, g, S, &tmap, Bnext, 0, lane);
        }
        if (PREP_NBUF == 2) buf ^= 1;
        b = bn;
    }
    // value range: warp -> CTA -> global (ordered-int encoding as k_resolve expects; NaN apart)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc.mx = fmaxf(acc.mx, __shfl_xor_sync(0xffffffffu, acc.mx, o));
        acc.mn = fminf(acc.mn, __shfl_xor_sync(0xffffffffu, acc.mn, o));
        acc.nan |= __shfl_xor_sync(0xffffffffu, acc.nan, o);
    }
    if (lane == 0) {
        if (acc.mx >= acc.mn) {   // the warp saw at least one non-NaN value
            atomicMax(&omx, f2ord(acc.mx));
            atomicMin(&omn, f2ord(acc.mn));
        }
        if (acc.nan) atomicOr(&cta_nan, 1u);
        if (nreg) atomicAdd(&cta_nreg, nreg);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (omn != 0xffffffffu) {
            atomicMax(&A.minmax[0], omx);
            atomicMax(&A.minmax[1], ~omn);
        }
        if (cta_nan) atomicOr(&A.minmax[2], 1u);
        if (cta_nreg) atomicAdd(&A.counters[0], cta_nreg);
    }
}

}  // namespace ftlz
