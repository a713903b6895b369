// blocks.cu -- per-block stages of pipeline.compress on B200 (sm_100a):
//   k_prep      stage (a)+(b): value range, input checksum, regression fit (numpy pairwise
//               order), sampled predictor selection                             (K0 + K1)
//   k_quant_reg stage (c) for regression blocks: one thread per block row      (K2, regression)
//   k_quant_lor stage (c) for Lorenzo blocks: one warp per block, plane wavefront (K2, Lorenzo)
//
// A CTA of k_prep / k_quant_reg owns a "pencil": P consecutive blocks along z inside one
// block row, whose rows are contiguous in memory.  The pencil is staged in shared memory
// with cp.async (LDGSTS, 16-byte chunks when the rows are 16-byte aligned), so a CTA keeps
// every load of its tile in flight at once.  Per-point index math is incremental (no integer
// division in the loops) and every float64 operation is an explicit __dadd_rn/__dmul_rn.

namespace ftlz {

// ------------------------------------------------------------------------------------------
// pencil geometry (host mirror in api.cu: pencil_cfg)
struct Pencil {
    long long bi, bj, bk0;
    int nblk;       // blocks in this pencil (<= P)
    int bx, by;     // extents shared by the pencil's blocks
    int bz_last;    // z extent of the last block
    int L;          // floats per row = (nblk - 1) * e + bz_last
};

FTLZ_DEV Pencil pencil_of(const Geom& g, u32 pid, int P, const FastDiv& fd_npz, const FastDiv& fd_cy) {
    Pencil Pn;
    u32 t = fdiv(pid, fd_npz);
    u32 pz = pid - t * fd_npz.d;
    u32 bi = fdiv(t, fd_cy);
    Pn.bi = bi;
    Pn.bj = t - bi * fd_cy.d;
    Pn.bk0 = (long long)pz * P;
    Pn.nblk = (int)min((long long)P, g.cz - Pn.bk0);
    Pn.bx = (Pn.bi == g.cx - 1) ? g.rx : g.e;
    Pn.by = (Pn.bj == g.cy - 1) ? g.ry : g.e;
    Pn.bz_last = (Pn.bk0 + Pn.nblk == g.cz) ? g.rz : g.e;
    Pn.L = (Pn.nblk - 1) * g.e + Pn.bz_last;
    return Pn;
}

FTLZ_DEV void cp_async16(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem));
}
FTLZ_DEV void cp_async4(void* smem, const void* gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gmem));
}
FTLZ_DEV void cp_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// issue the cp.async copies of a pencil tile: the CTA's threads cover (row, chunk) items,
// chunk = 16 bytes when the rows are 16-byte aligned (vec) else 4 bytes.
// tile[row * stride + z], row = i * by + j, z in [0, L).  Caller commits / waits.
FTLZ_DEV void issue_pencil(const float* __restrict__ x, const Geom& g, const Pencil& Pn, float* tile, int stride,
                           const FastDiv& fd_by, const PencilIO& io, int P) {
    const FastDiv& fp = (Pn.bk0 + Pn.nblk < g.cz) ? io.per_full : io.per_last;
    int per = (int)fp.d;
    int nrows = Pn.bx * Pn.by;
    long long base = ((Pn.bi * g.e) * g.ny + Pn.bj * g.e) * g.nz + Pn.bk0 * g.e;
    int c4 = io.vec ? (Pn.L >> 2) : 0;
    for (int t = threadIdx.x; t < nrows * per; t += blockDim.x) {
        int r = (int)fdiv((u32)t, fp), c = t - r * per;
        int i = (int)fdiv((u32)r, fd_by), j = r - i * Pn.by;
        const float* row = x + base + ((long long)i * g.ny + j) * g.nz;
        float* dst = tile + r * stride;
        if (c < c4) cp_async16(dst + 4 * c, row + 4 * c);
        else {
            int z = 4 * c4 + (c - c4);
            cp_async4(dst + z, row + z);
        }
    }
}
FTLZ_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
FTLZ_DEV void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
FTLZ_DEV void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

FTLZ_DEV void load_pencil(const float* __restrict__ x, const Geom& g, const Pencil& Pn, float* tile, int stride,
                          const FastDiv& fd_by, const PencilIO& io, int P) {
    issue_pencil(x, g, Pn, tile, stride, fd_by, io, P);
    cp_commit();
    cp_wait0();
}

// element p (row-major in block) -> tile address, incremental walker
struct TileWalk {
    int i, j, k, bx, by, bz, stride, zoff;
    int bye;  // tile rows per i (== by for pencil tiles, == e for per-block TMA tiles)
    FTLZ_DEV void set(int p) {
        int byz = by * bz;
        i = p / byz;
        int rem = p - i * byz;
        j = rem / bz;
        k = rem - j * bz;
    }
    FTLZ_DEV int addr() const { return (i * bye + j) * stride + zoff + k; }
    FTLZ_DEV void advance(int d) {  // p += d
        k += d;
        while (k >= bz) {
            k -= bz;
            if (++j >= by) { j = 0; i++; }
        }
    }
};

// warp-cooperative single-word correction (checksum.py:109-142) over a block held in the
// tile (element p at TileWalk address); 0 clean, 1 corrected, 2 uncorrectable
FTLZ_DEV void tile_checksum(const float* tile, TileWalk w0, int vol, int lane, u64* s, u64* si) {
    u64 a = 0, c = 0;
    TileWalk w = w0;
    w.set(lane);
    for (int p = lane; p < vol; p += 32) {
        u64 v = __float_as_uint(tile[w.addr()]);
        a += v;
        c += (u64)p * v;
        w.advance(32);
    }
    *s = warp_sum_u64(a);
    *si = warp_sum_u64(c);
}

FTLZ_DEV int tile_correct(float* tile, TileWalk w0, int vol, u64 st_s, u64 st_si, int lane) {
    u64 s, si;
    tile_checksum(tile, w0, vol, lane, &s, &si);
    if (s == st_s && si == st_si) return 0;
    u64 ds = s - st_s, dsi = si - st_si;
    if (ds == 0) return 2;
    for (int j0 = 0; j0 < vol; j0 += 32) {
        int jj = j0 + lane;
        bool cand = jj < vol && (u64)jj * ds == dsi;
        unsigned m = __ballot_sync(0xffffffffu, cand);
        while (m) {
            int l = __ffs(m) - 1;
            m &= m - 1;
            TileWalk w = w0;
            w.set(j0 + l);
            int ad = w.addr();
            u64 old = __float_as_uint(tile[ad]);
            u64 restored = old - ds;
            if (restored >> 32) continue;
            __syncwarp();
            if (lane == 0) tile[ad] = __uint_as_float((u32)restored);
            __syncwarp();
            u64 s2, si2;
            tile_checksum(tile, w0, vol, lane, &s2, &si2);
            if (s2 == st_s && si2 == st_si) return 1;
            __syncwarp();
            if (lane == 0) tile[ad] = __uint_as_float((u32)old);
            __syncwarp();
        }
    }
    return 2;
}

// apply the block's INPUT faults to its tile region (one lane); returns true if any
FTLZ_DEV bool apply_input_faults(const CompArgs& A, long long b, float* tile, TileWalk w0, int lane) {
    if (!A.n_faults) return false;
    int f0 = A.fault_first[b];
    if (f0 < 0) return false;
    bool any = false;
    for (int f = f0; f < A.n_faults && A.faults[f].block == b; f++) {
        if (A.faults[f].target != FTLZ_FAULT_INPUT) continue;
        any = true;
        if (lane == 0) {
            TileWalk w = w0;
            w.set((int)A.faults[f].element);
            int ad = w.addr();
            tile[ad] = __uint_as_float(__float_as_uint(tile[ad]) ^ (1u << A.faults[f].bit));
        }
    }
    __syncwarp();
    return any;
}

// ==========================================================================================
// K1: stage (a) + (b).  CTA = pencil, warp = block.
__global__ void __launch_bounds__(512) k_prep(CompArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = A.g;
    int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    Pencil Pn = pencil_of(g, blockIdx.x, A.P, A.fd_npz, A.fd_cy);
    float* tile = (float*)smem;
    int vmax = g.vmax;
    int nls = vmax / 64 + 8;
    double* wslot = (double*)(smem + A.tile_bytes) + (size_t)warp * (4 * nls + 2 * (vmax / 8 + 8) + 3 * 64);
    double* leafval = wslot;
    double* ar = leafval + 4 * nls;
    double* al = ar + (vmax / 8 + 8);
    double* cv = al + (vmax / 8 + 8);  // c tables: [0..63] i - hx, [64..127] j - hy, [128..191] k - hz
    __shared__ u32 cta_max, cta_min, cta_nan, cta_nreg;
    if (tid == 0) { cta_max = 0; cta_min = 0xffffffffu; cta_nan = 0; cta_nreg = 0; }
    load_pencil(A.x, g, Pn, tile, A.tile_stride, Pn.by == g.e ? A.fd_e : A.fd_ry, A.pio, A.P);
    __syncthreads();
    if (warp < Pn.nblk) {
        long long b = ((Pn.bi * g.cy) + Pn.bj) * g.cz + Pn.bk0 + warp;
        int bx = Pn.bx, by = Pn.by, bz = (warp == Pn.nblk - 1) ? Pn.bz_last : g.e;
        int vol = bx * by * bz;
        int xid = ((bx != g.e) ? 4 : 0) | ((by != g.e) ? 2 : 0) | ((bz != g.e) ? 1 : 0);
        const ExtPlan& PL = A.plans[xid];
        TileWalk w0;
        w0.bx = bx; w0.by = by; w0.bz = bz; w0.stride = A.tile_stride; w0.zoff = warp * g.e; w0.bye = by;
        double hx = (double)(bx - 1) / 2.0, hy = (double)(by - 1) / 2.0, hz = (double)(bz - 1) / 2.0;
        for (int t = lane; t < 64; t += 32) {
            cv[t] = __dadd_rn(int_to_f64(t), -hx);
            cv[64 + t] = __dadd_rn(int_to_f64(t), -hy);
            cv[128 + t] = __dadd_rn(int_to_f64(t), -hz);
        }
        __syncwarp();
        // ---- pass over every element exactly once: pairwise chains of S(v), S(ci v), S(cj v),
        //      S(ck v) (predict.py:81-104), plus checksum (checksum.py:171-181) and value range
        u32 mx = 0, mn = 0xffffffffu, nan = 0;
        u64 cs = 0, csi = 0;
        auto visit = [&](int p, const TileWalk& w, double t[4]) {
            float f = tile[w.addr()];
            u32 u = __float_as_uint(f);
            cs += u;
            csi += (u64)p * u;
            if (f != f) nan = 1;
            else {
                u32 o = f2ord(f);
                mx = max(mx, o);
                mn = min(mn, o);
            }
            double v = (double)f;
            t[0] = v;
            t[1] = __dmul_rn(cv[w.i], v);
            t[2] = __dmul_rn(cv[64 + w.j], v);
            t[3] = __dmul_rn(cv[128 + w.k], v);
        };
        double sums[4];
        if (vol < 8) {
            if (lane == 0) {
                double r[4] = {0.0, 0.0, 0.0, 0.0};
                TileWalk w = w0;
                w.set(0);
                for (int p = 0; p < vol; p++) {
                    double t[4];
                    visit(p, w, t);
#pragma unroll
                    for (int q = 0; q < 4; q++) r[q] = __dadd_rn(r[q], t[q]);
                    w.advance(1);
                }
#pragma unroll
                for (int q = 0; q < 4; q++) sums[q] = __dadd_rn(0.0, r[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; q++) sums[q] = __shfl_sync(0xffffffffu, sums[q], 0);
        } else {
            const Leaf* leaves = A.leaves + PL.leaf_off;
            int nchains = PL.nleaf * 8;
            for (int c0 = 0; c0 < nchains; c0 += 32) {
                int c = c0 + lane;
                int leaf = c >> 3, j8 = c & 7;
                double r[4] = {0.0, 0.0, 0.0, 0.0};
                int start = 0, len = 0;
                if (c < nchains) {
                    Leaf Lf = leaves[leaf];
                    start = Lf.start;
                    len = Lf.len;
                    int len8 = len - (len & 7);
                    TileWalk w = w0;
                    w.set(start + j8);
                    visit(start + j8, w, r);
                    for (int p = start + j8 + 8; p < start + len8; p += 8) {
                        w.advance(8);
                        double t[4];
                        visit(p, w, t);
#pragma unroll
                        for (int q = 0; q < 4; q++) r[q] = __dadd_rn(r[q], t[q]);
                    }
                }
#pragma unroll
                for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        double other = __shfl_xor_sync(0xffffffffu, r[q], o);
                        r[q] = (j8 & o) ? __dadd_rn(other, r[q]) : __dadd_rn(r[q], other);
                    }
                }
                if (j8 == 0 && c < nchains) {
                    int len8 = len - (len & 7);
                    if (len8 < len) {
                        TileWalk w = w0;
                        w.set(start + len8);
                        for (int p = start + len8; p < start + len; p++) {
                            double t[4];
                            visit(p, w, t);
#pragma unroll
                            for (int q = 0; q < 4; q++) r[q] = __dadd_rn(r[q], t[q]);
                            w.advance(1);
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 4; q++) leafval[leaf * 4 + q] = r[q];
                }
            }
            __syncwarp();
            if (lane == 0) {
                double stk[24][4];
                int sp = 0;
                for (int l = 0; l < PL.nleaf; l++) {
#pragma unroll
                    for (int q = 0; q < 4; q++) stk[sp][q] = leafval[l * 4 + q];
                    sp++;
                    for (int t = 0; t < leaves[l].ncomb; t++) {
#pragma unroll
                        for (int q = 0; q < 4; q++) stk[sp - 2][q] = __dadd_rn(stk[sp - 2][q], stk[sp - 1][q]);
                        sp--;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; q++) sums[q] = __dadd_rn(0.0, stk[0][q]);
            }
#pragma unroll
            for (int q = 0; q < 4; q++) sums[q] = __shfl_sync(0xffffffffu, sums[q], 0);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            nan |= __shfl_xor_sync(0xffffffffu, nan, o);
        }
        cs = warp_sum_u64(cs);
        csi = warp_sum_u64(csi);
        if (lane == 0) {
            atomicMax(&cta_max, mx);
            atomicMin(&cta_min, mn);
            atomicOr(&cta_nan, nan);
        }
        // ---- coefficients (batch form, predict.py:90-104)
        float4 cf;
        {
            double out0 = __ddiv_rn(sums[0], (double)vol);
            double sl[3];
            int ext[3] = {bx, by, bz};
#pragma unroll
            for (int ax = 0; ax < 3; ax++) {
                int e = ext[ax];
                if (e == 1) { sl[ax] = 0.0; continue; }
                double denom = __ddiv_rn((double)((long long)vol * ((long long)e * e - 1)), 12.0);
                sl[ax] = __ddiv_rn(sums[ax + 1], denom);
                out0 = __dadd_rn(out0, -__ddiv_rn(__dmul_rn(sl[ax], (double)(e - 1)), 2.0));
            }
            cf = make_float4(__double2float_rn(out0), __double2float_rn(sl[0]), __double2float_rn(sl[1]),
                             __double2float_rn(sl[2]));
        }
        // ---- hooks after stage (a): COEFFS_FITTED, INPUT_AFTER_CHECKSUM (pipeline.py:328-329)
        bool bad = false;
        if (A.n_faults && A.fault_first[b] >= 0) {
            int f0 = A.fault_first[b];
            for (int f = f0; f < A.n_faults && A.faults[f].block == b; f++)
                if (A.faults[f].target == FTLZ_FAULT_COEFF) {
                    float* c4 = (float*)&cf;
                    c4[A.faults[f].element] = __uint_as_float(__float_as_uint(c4[A.faults[f].element]) ^ (1u << A.faults[f].bit));
                }
            if (apply_input_faults(A, b, tile, w0, lane) && A.protect_input) {
                // stage (b) verification against the stage (a) checksum (pipeline.py:331-361)
                int r = tile_correct(tile, w0, vol, cs, csi, lane);
                if (r == 1 && lane == 0) { A.events[b] |= 1; atomicAdd(&A.counters[3], 1u); }
                if (r == 2) {
                    bad = true;
                    if (lane == 0) { A.events[b] |= 4; atomicAdd(&A.counters[3], 1u); }
                }
            }
            __syncwarp();
        }
        if (!bad) {
            // ---- sampled selection (predict.py:196-231)
            int ns = PL.ns;
            double c0 = (double)cf.x, c1 = (double)cf.y, c2 = (double)cf.z, c3 = (double)cf.w;
            int byz = by * bz;
            TileWalk w = w0;
            if (ns > 0) w.set(8 * (lane + 1));
            for (int q = lane; q < ns; q += 32) {
                int i = w.i, j = w.j, k = w.k;
                int ad = w.addr();
                double v = (double)tile[ad];
                double pr = __dadd_rn(__dadd_rn(__dadd_rn(c0, __dmul_rn(c1, int_to_f64(i))), __dmul_rn(c2, int_to_f64(j))),
                                      __dmul_rn(c3, int_to_f64(k)));
                int sr = A.tile_stride, sp = by * sr;  // tile offsets of (i-1) and (j-1)
                double d100 = i > 0 ? (double)tile[ad - sp] : 0.0;
                double d010 = j > 0 ? (double)tile[ad - sr] : 0.0;
                double d001 = k > 0 ? (double)tile[ad - 1] : 0.0;
                double d110 = (i > 0 && j > 0) ? (double)tile[ad - sp - sr] : 0.0;
                double d101 = (i > 0 && k > 0) ? (double)tile[ad - sp - 1] : 0.0;
                double d011 = (j > 0 && k > 0) ? (double)tile[ad - sr - 1] : 0.0;
                double d111 = (i > 0 && j > 0 && k > 0) ? (double)tile[ad - sp - sr - 1] : 0.0;
                double pl = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(d100, d010), d001), -d110), -d101), -d011), d111);
                ar[q] = fabs(__dadd_rn(v, -pr));
                al[q] = fabs(__dadd_rn(v, -pl));
                w.advance(256);
                (void)byz;
            }
            __syncwarp();
            double e2[2];
            if (ns < 8) {
                if (lane == 0) {
                    double r0 = 0.0, r1 = 0.0;
                    for (int q = 0; q < ns; q++) { r0 = __dadd_rn(r0, ar[q]); r1 = __dadd_rn(r1, al[q]); }
                    e2[0] = __dadd_rn(0.0, r0);
                    e2[1] = __dadd_rn(0.0, r1);
                }
                e2[0] = __shfl_sync(0xffffffffu, e2[0], 0);
                e2[1] = __shfl_sync(0xffffffffu, e2[1], 0);
            } else {
                warp_pairwise<2>(A.leaves + PL.sleaf_off, PL.nsleaf, ns,
                                 [&](int q, double* t) { t[0] = ar[q]; t[1] = al[q]; }, leafval, e2, lane);
            }
            double er = e2[0], el = e2[1];
            if (A.n_faults && A.fault_first[b] >= 0) {
                int f0 = A.fault_first[b];
                for (int f = f0; f < A.n_faults && A.faults[f].block == b; f++) {
                    if (A.faults[f].target != FTLZ_FAULT_ESTIMATE) continue;
                    u64 bit = 1ull << A.faults[f].bit;
                    if (A.faults[f].element == 0) er = __longlong_as_double((long long)(dbits(er) ^ bit));
                    else el = __longlong_as_double((long long)(dbits(el) ^ bit));
                }
            }
            int kind = er < el ? 1 : 0;
            if (A.override_ && A.override_[b] >= 0) kind = A.override_[b];
            if (lane == 0) {
                A.coef[b] = cf;
                A.insum[b] = cs;
                A.inisum[b] = csi;
                A.ind[b] = (u8)kind;
                if (kind == 1) atomicAdd(&cta_nreg, 1u);
                else A.lor_list[atomicAdd(&A.counters[4], 1u)] = (u32)b;
            }
        } else if (lane == 0) {
            A.ind[b] = 0;
            A.coef[b] = cf;
        }
    }
    __syncthreads();
    if (tid == 0) {
        atomicMax(&A.minmax[0], cta_max);
        atomicMax(&A.minmax[1], ~cta_min);
        if (cta_nan) atomicOr(&A.minmax[2], 1u);
        if (cta_nreg) atomicAdd(&A.counters[0], cta_nreg);
    }
}

// ==========================================================================================
// emit pass (both predictors), warp = block, row-major order: unpredictable words, bins
// checksum, warp-aggregated histogram, bins to the encoder layout
FTLZ_DEV void emit_block(const CompArgs& A, long long b, int vol, const u16* bins16, const float* tile,
                         TileWalk w0, u64 dcsum, int lane, u32* hwin, int wlo) {
    const Geom& g = A.g;
    u64 bs = 0, bis = 0;
    u32 nunp = 0;
    u32* unp = A.unp_scratch + (size_t)b * g.vmax;
    size_t bidx0 = bins_index(g, b, 0);
    TileWalk w = w0;
    w.set(lane);
    for (int p0 = 0; p0 < vol; p0 += 32) {
        int p = p0 + lane;
        bool act = p < vol;
        int bin = act ? bins16[p] : -1;
        unsigned zm = __ballot_sync(0xffffffffu, bin == 0);
        if (bin == 0) unp[nunp + __popc(zm & ((1u << lane) - 1u))] = __float_as_uint(tile[w.addr()]);
        nunp += __popc(zm);
        if (act) {
            bs += (u64)bin;
            bis += (u64)p * (u64)bin;
            // [group][chunk][lane][8]: chunk p/8 advances 256 elements per 8 points
            A.bins[bidx0 + (size_t)(p >> 3) * 256 + (p & 7)] = (u16)bin;
        }
        unsigned peers = __match_any_sync(0xffffffffu, bin);
        if (act && lane == __ffs(peers) - 1) hist_add(hwin, A.hist, wlo, bin, (u32)__popc(peers));
        w.advance(32);
    }
    dcsum = warp_sum_u64(dcsum);
    bs = warp_sum_u64(bs);
    bis = warp_sum_u64(bis);
    if (lane == 0) {
        A.unpc[b] = nunp;
        if (nunp) atomicAdd((u64*)&A.layout[LAYOUT_NUNP], (u64)nunp);
        A.bsum[b] = bs;
        A.bisum[b] = bis;
        A.dcs[b] = dcsum;
    }
}

// 2-of-3 voting on scalars (pipeline.py:157-179); eval3 only on mismatch
struct DupPred {
    double v;
    bool mismatch, disagree;
};
template <typename F3>
FTLZ_DEV DupPred vote(double a, double b, F3 eval3) {
    DupPred r;
    r.v = a;
    r.mismatch = false;
    r.disagree = false;
    if (dbits(a) == dbits(b)) return r;
    double c = eval3();
    r.mismatch = true;
    bool ac = dbits(a) == dbits(c), bc = dbits(b) == dbits(c);
    r.v = ac ? a : b;
    r.disagree = !(bc || ac);
    return r;
}

// one point of stage (c) given its prediction(s): returns bin, writes reconstructed value
// (pipeline.py:390-409 / 416-438; quantize.py:37-100)
template <typename F3P>
FTLZ_DEV int quant_point(const QuantParams& Q, float x32, double p1, double p2, bool dup, F3P pred3,
                         float* r32, bool* mism, double* back_out) {
    double x64 = (double)x32;
    double pred = p1;
    bool pdis = false;
    if (dup && dbits(p1) != dbits(p2)) {
        DupPred pr = vote(p1, p2, pred3);
        pred = pr.v;
        pdis = pr.disagree;
        *mism = true;
    }
    bool ok;
    int bin = quantize(Q, __dadd_rn(x64, -pred), &ok);
    if (pdis) ok = false;
    double offs = int_to_f64(bin - Q.center);
    double d1 = __dadd_rn(pred, __dmul_rn(Q.twoeb, offs));
    if (dup) {
        double d2 = __dadd_rn(opaque(pred), __dmul_rn(Q.twoeb, opaque(offs)));
        if (dbits(d1) != dbits(d2)) {
            DupPred dr = vote(d1, d2, [&] { return __dadd_rn(pred, __dmul_rn(Q.twoeb, opaque(opaque(offs)))); });
            d1 = dr.v;
            if (dr.disagree) ok = false;
            *mism = true;
        }
    }
    float d32 = __double2float_rn(d1);
    double back = (double)d32;
    bool keep = ok && fabs(__dadd_rn(x64, -back)) <= Q.eb;
    *r32 = keep ? d32 : x32;
    *back_out = keep ? back : x64;
    return keep ? bin : 0;
}

// ==========================================================================================
// K2 (Lorenzo blocks): warp = block from the Lorenzo list; constant-(i+j+k) wavefront over a
// float64 buffer of reconstructed values (pipeline.py:199-213, 410-438)
__global__ void __launch_bounds__(128) k_quant_lor(CompArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geom& g = A.g;
    if (dev_failed(A.st)) return;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    unsigned char* slot = smem + (size_t)warp * A.lor_slot;
    float* xf = (float*)slot;
    double* xd = (double*)(slot + (((size_t)g.vmax * 4 + 15) & ~(size_t)15));
    u16* bins16 = (u16*)(xd + g.vmax);
    u32* hwin = (u32*)(smem + (size_t)nw * A.lor_slot);
    const int wlo = A.center - HWIN / 2;
    for (int t = threadIdx.x; t < HWIN; t += blockDim.x) hwin[t] = 0;
    __syncthreads();
    const QuantParams Q = *A.qp;
    u32 n = A.counters[4];
    bool dup = A.dup_eval != 0;
    for (long long idx = (long long)blockIdx.x * nw + warp; idx < (long long)n; idx += (long long)gridDim.x * nw) {
        long long b = A.lor_list[idx];
        if (A.events[b] & 4) continue;
        BlockInfo B = block_info(g, b);
        int vol = B.vol, bz = B.bz, byz = B.by * B.bz;
        // stage the block (rows of bz floats) with cp.async
        long long base = ((B.bi * g.e) * g.ny + B.bj * g.e) * g.nz + B.bk * g.e;
        {
            TileWalk w;
            w.bx = B.bx; w.by = B.by; w.bz = bz; w.stride = 0; w.zoff = 0; w.bye = B.by;
            w.set(lane);
            for (int p = lane; p < vol; p += 32) {
                cp_async4(xf + p, A.x + base + ((long long)w.i * g.ny + w.j) * g.nz + w.k);
                w.advance(32);
            }
            cp_async_wait();
        }
        __syncwarp();
        TileWalk w0;
        w0.bx = B.bx; w0.by = B.by; w0.bz = bz; w0.stride = bz * B.by; w0.zoff = 0; w0.bye = B.by;
        // block-local layout: addr = (i*by + j)*bz + k  (stride = bz per row with by rows)
        w0.stride = bz;
        if (!A.protect_input) apply_input_faults(A, b, xf, w0, lane);
        else {
            int r = tile_correct(xf, w0, vol, A.insum[b], A.inisum[b], lane);
            if (r == 1 && lane == 0) { A.events[b] |= 1; atomicAdd(&A.counters[3], 1u); }
            if (r == 2) {
                if (lane == 0) { A.events[b] |= 4; atomicAdd(&A.counters[3], 1u); }
                continue;
            }
        }
        __syncwarp();
        const ExtPlan& PL = A.plans[B.xid];
        const u32* crd = A.coords + PL.coord_off;
        const u32* wave = A.wave + PL.wave_off;
        const u32* planes = A.planes + PL.plane_off;
        bool mism = false;
        u64 dcsum = 0;
        for (int s = 0; s < PL.nplanes; s++) {
            int q0 = __ldg(planes + s), q1 = __ldg(planes + s + 1);
            for (int q = q0 + lane; q < q1; q += 32) {
                int p = __ldg(wave + q);
                u32 c = __ldg(crd + p);
                int i = c & 0xff, j = (c >> 8) & 0xff, k = c >> 16;
                double d100 = i > 0 ? xd[p - byz] : 0.0;
                double d010 = j > 0 ? xd[p - bz] : 0.0;
                double d001 = k > 0 ? xd[p - 1] : 0.0;
                double d110 = (i > 0 && j > 0) ? xd[p - byz - bz] : 0.0;
                double d101 = (i > 0 && k > 0) ? xd[p - byz - 1] : 0.0;
                double d011 = (j > 0 && k > 0) ? xd[p - bz - 1] : 0.0;
                double d111 = (i > 0 && j > 0 && k > 0) ? xd[p - byz - bz - 1] : 0.0;
                auto lor = [&](double first) {
                    return __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(first, d010), d001), -d110), -d101), -d011), d111);
                };
                double p1 = lor(d100);
                double p2 = dup ? lor(opaque(d100)) : p1;
                float r32;
                double back;
                int bin = quant_point<>(Q, xf[p], p1, p2, dup, [&] { return lor(opaque(opaque(d100))); }, &r32, &mism, &back);
                xd[p] = back;
                bins16[p] = (u16)bin;
                dcsum += __float_as_uint(r32);
            }
            __syncwarp();
        }
        if (__ballot_sync(0xffffffffu, mism) && lane == 0) atomicOr(&A.counters[1], 1u << (B.xid * 2 + 0));
        emit_block(A, b, vol, bins16, xf, w0, dcsum, lane, hwin, wlo);
        __syncwarp();
    }
    __syncthreads();
    hist_flush(hwin, A.hist, wlo, A.cap);
}

}  // namespace ftlz
