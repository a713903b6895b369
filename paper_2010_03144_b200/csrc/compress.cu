// compress.cu -- device side of pipeline.compress (pipeline.py:287-537) + container.serialize
// (container.py:109-147) for B200 (sm_100a).
//
// Kernel sequence (one stream, no host sync until the report read-back):
//   k_prep      (prep_block.cu) stage (a)+(b): value range, input checksums, regression fit with numpy's
//               pairwise float64 summation order, sampled predictor selection   (K0+K1)
//   k_resolve   resolved error bound (core.py:182-193) + quantizer constants
//   k_quant_*   (quant_block.cu, blocks.cu) stage (c): verify input, predict (duplicated), quantize, reconstruct
//               (duplicated), double-check, bins/unpredictables/checksums/sum_dc/histogram (K2)
//   k_fault_bins  bins-stage faults: verify/correct (protect_bins) and histogram fix-up
//   k_codebook  canonical Huffman codebook from the global histogram (K3), archive layout
//   k_enc_*     (encode.cu) per-block bit lengths, block offsets, MSB-first packing (K4)
//   k_assemble  header, block table, unpredictable words, sum_dc section (K5)
#include <cstdio>

#include "common.cuh"
#include "tma.cuh"

namespace ftlz {

// ------------------------------------------------------------------------------------------
// workspace pointers for one compress call (carved by the host from one allocation)
struct CompArgs {
    Geom g;
    const float* x;
    int protect_input, protect_bins, dup_eval, store_sum_dc;
    int eb_mode;
    double eb_value;
    int cap, center;
    FastDiv fd_e, fd_ry, fd_rz;   // launch-constant divisors (row decomposition)
    StageCfg stage;           // per-block TMA tiles (k_quant_reg)
    int qr_slot, qr_tab;      // k_quant_reg: smem bytes per warp, offset of the row tables in a slot
    int rmax;                 // rows per block (max)
    int pp_slot, pp_nls, pp_ns;   // k_prep: smem bytes per warp, leaf / sample slots
    int dbg;                  // debugging switches (FTLZ_DBG)
    int lor_slot;             // smem bytes per warp in k_quant_lor
    int r10, r10_slot;        // k_quant_reg10 active (edge 10, TMA tiles of 12-float rows); smem per warp
    int lor_fused, pad_lf;    // k_quant_reg10 also quantizes the Lorenzo blocks (no k_quant_lor launch)
    int lor2d, pad_l2;        // 2-D Lorenzo blocks by k_quant_lor2d; k_quant_lor takes defer_list (counters[9])
    u32* defer_list;
    u32* lor_list;            // Lorenzo blocks (appended by k_prep)
    u32* r10_list;            // regression blocks for k_quant_reg10 (k_reglist; counters[5] entries)
    u32* regx_list;           // the other regression blocks, for k_quant_reg (counters[6] entries)
    int n_faults;
    const ftlz_fault* faults;    // device copy
    const int* fault_first;      // nb: first fault index of this block or -1 (faults sorted by block)
    const int8_t* override_;     // nb or null
    const ExtPlan* plans;        // 8 entries
    const Leaf* leaves;
    const u32* coords;
    const u32* wave;
    const u32* wcrd;     // coordinates in wavefront order
    const u32* planes;
    // per-block
    float4* coef;
    u64* insum;
    u64* inisum;
    u8* ind;
    u32* unpc;
    u64* bsum;
    u64* bisum;
    u64* dcs;
    u32* bitlen;
    u32* lanepre;        // nb x 32: bit offset of each lane's symbol range inside its block
    u64* bitoff;         // nb: payload bit offset of each block
    u32* regpre;
    u64* unppre;
    u8* events;          // bit0 input corrected, bit1 bins corrected, bit2 input uncorrectable, bit3 bins uncorrectable
    // globals
    DevStatus* st;
    u32* minmax;         // [0] ordered max, [1] ordered min, [2] nan flag
    u32* counters;       // [0] n_reg, [1] dup group flags, [2] encode ticket, [3] events, [4] n_lor
    QuantParams* qp;
    u64* hist;           // cap entries (u64: a field may hold more than 2^32 points)
    u64* enc;            // cap entries: code << 6 | len (0 = absent)
    u64* layout;         // archive layout (see LAYOUT_*)
    long long pb0, pb1;  // k_prep's blocks (slabs of block layers when the upload is overlapped)
    u64* lookback;       // encode tiles
    u16* bins;
    u32* unp_scratch;    // nb * vmax (sparse)
    u8* out;
    u64 out_cap;
    double* dscratch;    // generic per-CTA scratch for big blocks (unused for e <= 16)
};

enum {
    LAYOUT_TABLE_LEN = 0, LAYOUT_BOOK_OFF, LAYOUT_NSYM, LAYOUT_PAYLEN_OFF, LAYOUT_PAY_OFF,
    LAYOUT_PAY_BYTES, LAYOUT_UNP_OFF, LAYOUT_NUNP, LAYOUT_SDC_OFF, LAYOUT_TOTAL, LAYOUT_TOTAL_BITS,
    LAYOUT_MAXLEN, LAYOUT_NREG, LAYOUT_EB_BITS, LAYOUT_SYMLO, LAYOUT_SYMHI, LAYOUT_COUNT
};

// ------------------------------------------------------------------------------------------
// numpy pairwise sums over a block: chains of 8 strided accumulators per leaf, combined with
// the exact tree ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), tail added sequentially, leaves combined
// by the host-built post-order program, and the 0.0 identity added last.
template <int NV, typename Getter>
FTLZ_DEV void warp_pairwise(const Leaf* leaves, int nleaf, int n, Getter get, double* leafval,
                            double out[NV], int lane) {
    if (n < 8) {
        // whole reduction below 8 elements: 0.0 then sequential (never split further)
        if (lane == 0) {
            double r[NV];
#pragma unroll
            for (int v = 0; v < NV; v++) r[v] = 0.0;
            for (int p = 0; p < n; p++) {
                double t[NV];
                get(p, t);
#pragma unroll
                for (int v = 0; v < NV; v++) r[v] = __dadd_rn(r[v], t[v]);
            }
#pragma unroll
            for (int v = 0; v < NV; v++) out[v] = __dadd_rn(0.0, r[v]);
        }
#pragma unroll
        for (int v = 0; v < NV; v++) out[v] = __shfl_sync(0xffffffffu, out[v], 0);
        return;
    }
    int nchains = nleaf * 8;
    for (int c0 = 0; c0 < nchains; c0 += 32) {
        int c = c0 + lane;
        int leaf = c >> 3, j = c & 7;
        double r[NV];
#pragma unroll
        for (int v = 0; v < NV; v++) r[v] = 0.0;
        int start = 0, len = 0;
        if (c < nchains) {
            Leaf L = leaves[leaf];
            start = L.start;
            len = L.len;
            int len8 = len - (len & 7);
            get(start + j, r);
            for (int p = start + j + 8; p < start + len8; p += 8) {
                double t[NV];
                get(p, t);
#pragma unroll
                for (int v = 0; v < NV; v++) r[v] = __dadd_rn(r[v], t[v]);
            }
        }
        // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) : lower lane is the left operand
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
#pragma unroll
            for (int v = 0; v < NV; v++) {
                double other = __shfl_xor_sync(0xffffffffu, r[v], o);
                r[v] = (j & o) ? __dadd_rn(other, r[v]) : __dadd_rn(r[v], other);
            }
        }
        if (j == 0 && c < nchains) {
            int len8 = len - (len & 7);
            for (int p = start + len8; p < start + len; p++) {
                double t[NV];
                get(p, t);
#pragma unroll
                for (int v = 0; v < NV; v++) r[v] = __dadd_rn(r[v], t[v]);
            }
#pragma unroll
            for (int v = 0; v < NV; v++) leafval[leaf * NV + v] = r[v];
        }
    }
    __syncwarp();
    if (lane == 0) {
        // post-order combine: stack of partial sums (depth <= log2(n/64) + 2)
        double stk[24][NV];
        int sp = 0;
        for (int l = 0; l < nleaf; l++) {
#pragma unroll
            for (int v = 0; v < NV; v++) stk[sp][v] = leafval[l * NV + v];
            sp++;
            int nc = leaves[l].ncomb;
            for (int t = 0; t < nc; t++) {
#pragma unroll
                for (int v = 0; v < NV; v++) stk[sp - 2][v] = __dadd_rn(stk[sp - 2][v], stk[sp - 1][v]);
                sp--;
            }
        }
#pragma unroll
        for (int v = 0; v < NV; v++) out[v] = __dadd_rn(0.0, stk[0][v]);
    }
#pragma unroll
    for (int v = 0; v < NV; v++) out[v] = __shfl_sync(0xffffffffu, out[v], 0);
}

// ==========================================================================================
// resolve the bound (core.py:182-193) and the quantizer constants
__global__ void k_resolve(CompArgs A) {
    double eb = A.eb_value;
    if (A.eb_mode == 1) {
        float mx = ord2f(A.minmax[0]), mn = ord2f(~A.minmax[1]);
        double range = A.minmax[2] ? __longlong_as_double(0x7ff8000000000000ll)
                                   : __dadd_rn((double)mx, -(double)mn);
        eb = __dmul_rn(A.eb_value, range);
    }
    QuantParams Q;
    Q.eb = eb;
    Q.twoeb = __dmul_rn(2.0, eb);
    Q.rcp = __ddiv_rn(1.0, Q.twoeb);
    Q.twoeb_dup = __dmul_rn(eb, 2.0);
    Q.cap = A.cap;
    Q.center = A.cap / 2;
    Q.capd2 = 2.0 * (double)A.cap;
    Q.capd2_bits = dbits(Q.capd2);
    Q.eb_bits = dbits(eb);
    u64 tb = dbits(Q.twoeb) & 0x7fffffffffffffffull, rb = dbits(Q.rcp) & 0x7fffffffffffffffull;
    bool normal = tb >= 0x0010000000000000ull && tb < 0x7ff0000000000000ull &&
                  rb >= 0x0010000000000000ull && rb < 0x7ff0000000000000ull;
    Q.exact_div = normal ? 0 : 1;
    Q.rcp32 = __double2float_rn(Q.rcp);
    Q.eb32 = __double2float_rn(eb);
    Q.band32 = Q.eb32 * 9.5367431640625e-07f;   // 2^-20
    Q.sbig = A.cap > 65536 ? (float)A.cap : 65536.0f;
    {
        // both float32 operands well inside the normal range (the error bounds assume it)
        const float ar = fabsf(Q.rcp32), ae = fabsf(Q.eb32);
        Q.fast32 = normal && ar >= 7.9e-31f && ar <= 1.2e30f && ae >= 7.9e-31f && ae <= 1.2e30f ? 1 : 0;
    }
    Q.pad2 = 0;
    *A.qp = Q;
    A.layout[LAYOUT_EB_BITS] = dbits(eb);
    if (!(eb > 0.0) || !(dbits(eb) < 0x7ff0000000000000ull)) {
        dev_fail(A.st, FTLZ_ERR_DEGENERATE_BOUND, FTLZ_K_DEGENERATE, -1, -1, 0, 0, 0);
        return;
    }
    // uncorrectable input from stage (b) -> first in extent-sorted group order is chosen
    // by the host from events (pipeline.py:342-345); flag it here
}

// ==========================================================================================
// K3: canonical Huffman codebook (encode.py:26-71) on one CTA.
// Two-queue merge over leaves sorted by (weight, symbol) reproduces the heap with
// (weight, tiebreak) keys exactly: leaf ties break by symbol rank, merged nodes are created
// in non-decreasing weight order and pop FIFO, and a leaf wins a weight tie against any
// merged node (its tiebreak < n <= every merged tiebreak).
#define CB_THREADS 1024
#define CB_SMEM_KEYS 8192

struct CodebookScratch {
    u64* keys;     // 2 * cap (sorted leaves; later (len, sym) keys)
    u32* syms;     // cap (sorted by weight order)
    u64* w;        // 2 * cap node weights (leaves then internal)
    u32* parent;   // 2 * cap
    u8* lens;      // cap (by symbol)
    u32* bm;       // (cap + 31) / 32 words: alphabet bitmap (k_cb_bitmap)
};

// two-queue Huffman merge over leaves sorted by (weight, symbol) (the reference heap with its
// (weight, tie) order, encode.py:26-71): leaves 0..n-1, merged nodes n..2n-2 in creation order,
// W[node] its weight.  Queue state: li leaves and (mi - n) merged nodes consumed, mk the next
// merged id.  cb_merge_seq runs up to `steps` merges from that state with the queue heads in
// registers.  W must point into one memory space (shared or global) so accesses stay typed.
template <typename WT, typename SetParent>
FTLZ_DEV void cb_merge_seq(WT* W, int n, int& li_, int& mi_, int& mk_, int steps, SetParent set_parent) {
    const WT INF = (WT)~(WT)0;
    int li = li_, mi = mi_, mk = mk_;
    WT L0 = li < n ? W[li] : INF, L1 = li + 1 < n ? W[li + 1] : INF;
    WT L2 = li + 2 < n ? W[li + 2] : INF, L3 = li + 3 < n ? W[li + 3] : INF;
    WT M0 = mi < mk ? W[mi] : INF, M1 = mi + 1 < mk ? W[mi + 1] : INF;
    WT M2 = mi + 2 < mk ? W[mi + 2] : INF, M3 = mi + 3 < mk ? W[mi + 3] : INF;
    const int mend = 2 * n - 1;
    for (int t = 0; t < steps && mk < mend; t++) {
        const bool c1 = L0 <= M0, c2 = L1 <= M0, c3 = L0 <= M1;
        const bool LL = c1 && c2, MM = !c1 && !c3;
        const int ca = MM ? mi : li, cb = LL ? li + 1 : (MM ? mi + 1 : mi);
        const WT sum = LL ? L0 + L1 : (MM ? M0 + M1 : L0 + M0);
        const int dl = LL ? 2 : (MM ? 0 : 1), dm = 2 - dl;
        const WT nl0 = li + 4 < n ? W[li + 4] : INF, nl1 = li + 5 < n ? W[li + 5] : INF;
        const WT nm0 = mi + 4 < mk ? W[mi + 4] : INF, nm1 = mi + 5 < mk ? W[mi + 5] : INF;
        const WT a0 = dl == 0 ? L0 : (dl == 1 ? L1 : L2), a1 = dl == 0 ? L1 : (dl == 1 ? L2 : L3);
        const WT a2 = dl == 0 ? L2 : (dl == 1 ? L3 : nl0), a3 = dl == 0 ? L3 : (dl == 1 ? nl0 : nl1);
        L0 = a0; L1 = a1; L2 = a2; L3 = a3;
        const WT b0 = dm == 0 ? M0 : (dm == 1 ? M1 : M2), b1 = dm == 0 ? M1 : (dm == 1 ? M2 : M3);
        const WT b2 = dm == 0 ? M2 : (dm == 1 ? M3 : nm0), b3 = dm == 0 ? M3 : (dm == 1 ? nm0 : nm1);
        li += dl;
        mi += dm;
        W[mk] = sum;
        const int q = mk - mi;   // merged nodes waiting before the new one
        M0 = q == 0 ? sum : b0;
        M1 = q == 1 ? sum : b1;
        M2 = q == 2 ? sum : b2;
        M3 = q == 3 ? sum : b3;
        set_parent(ca, mk);
        set_parent(cb, mk);
        mk++;
    }
    li_ = li; mi_ = mi; mk_ = mk;
}

// the same merge, round-synchronous on the whole CTA.  With y1 <= y2 <= ... the remaining nodes
// in (weight, tie) order and s1 = y1 + y2, the heap pops the pairs (y1, y2), (y3, y4), ...
// as long as y_2j precedes s1: s1 is the newest node (largest tie), so that is w(y_2j) <= w(s1),
// and the merged sums are non-decreasing, so they join the merged queue in order.  A round
// merges k = floor(#{y : w(y) <= w(s1)} / 2) pairs at once (c4: 4890 leaves in 23 rounds);
// rounds with fewer than CB_KMIN pairs run CB_SEQ sequential merges instead (one thread).
#define CB_KMIN 32
#define CB_SEQ 64
template <typename WT, typename SetParent>
FTLZ_DEV void cb_merge_par(WT* W, int n, SetParent set_parent) {
    __shared__ int s_li, s_mi, s_mk, s_k, s_a;
    const int tid = threadIdx.x;
    if (tid == 0) { s_li = 0; s_mi = n; s_mk = n; }
    __syncthreads();
    // number of leaves among the first d remaining nodes (leaves win weight ties)
    auto split = [&](int li, int llen, int mi, int mlen, int d) {
        int lo = max(0, d - mlen), hi = min(d, llen);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (W[li + mid] <= W[mi + d - 1 - mid]) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    // first index in [lo, hi) with W > v
    auto upper = [&](int lo, int hi, WT v) {
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (W[mid] <= v) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    const int mend = 2 * n - 1;
    while (true) {
        const int li = s_li, mi = s_mi, mk = s_mk;
        __syncthreads();   // the state is read before thread 0 moves it
        if (mk >= mend) break;
        const int llen = n - li, mlen = mk - mi;
        if (tid == 0) {
            // s1 from the two smallest remaining nodes
            int x = 0, y = 0;
            WT s1 = 0;
            for (int u = 0; u < 2; u++) {
                const bool tl = x < llen && (y >= mlen || W[li + x] <= W[mi + y]);
                s1 += tl ? W[li + x] : W[mi + y];
                x += tl;
                y += !tl;
            }
            const int c = (upper(li, n, s1) - li) + (upper(mi, mk, s1) - mi);
            const int k = c >> 1;
            if (k < CB_KMIN) {
                int l2 = li, m2 = mi, k2 = mk;
                cb_merge_seq(W, n, l2, m2, k2, CB_SEQ, set_parent);
                s_li = l2; s_mi = m2; s_mk = k2; s_k = 0;
            } else {
                s_k = k;
                s_a = split(li, llen, mi, mlen, 2 * k);
            }
        }
        __syncthreads();
        const int k = s_k;
        if (k) {
            for (int j = tid; j < k; j += blockDim.x) {
                const int d = 2 * j;
                int x = split(li, llen, mi, mlen, d), y = d - x;
                int id[2];
                WT w[2];
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const bool tl = x < llen && (y >= mlen || W[li + x] <= W[mi + y]);
                    id[u] = tl ? li + x : mi + y;
                    w[u] = W[id[u]];
                    x += tl;
                    y += !tl;
                }
                W[mk + j] = w[0] + w[1];
                set_parent(id[0], mk + j);
                set_parent(id[1], mk + j);
            }
            __syncthreads();
            if (tid == 0) { s_li = li + s_a; s_mi = mi + 2 * k - s_a; s_mk = mk + k; }
        }
        __syncthreads();
    }
}

// alphabet bitmap {0} U {s : hist[s] > 0} over the whole grid: the histogram is read once by
// all SMs instead of by k_codebook's single CTA (a warp per 32-symbol word, coalesced)
__global__ void __launch_bounds__(256) k_cb_bitmap(CompArgs A, u32* bm) {
    if (dev_failed(A.st)) return;
    const int lane = threadIdx.x & 31;
    const int w = (int)(blockIdx.x * 8 + (threadIdx.x >> 5));
    const int sy = w * 32 + lane;
    if (w * 32 >= A.cap) return;
    const u32 m = __ballot_sync(0xffffffffu, sy < A.cap && (sy == 0 || A.hist[sy] != 0u));
    if (lane == 0) bm[w] = m;
}

// one stable LSD counting pass of the whole CTA: out = in ordered by the digit
// (key >> shift) & (2^RBITS - 1), equal digits in input order.  Warp w owns a contiguous run of
// 32-item steps; a step ranks its lanes by __match_any_sync on the digit, and per-warp digit
// counters (cnt: nwarps x 2^RBITS words) give every item its slot (count, offsets, scatter).
template <int RBITS>
FTLZ_DEV void cb_radix_pass(const u64* in, u64* out, int n, int shift, u32* cnt, u32* base) {
    constexpr int R = 1 << RBITS;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int steps = (n + 32 * nw - 1) / (32 * nw);
    const int i0 = warp * steps * 32;
    u32* wc = cnt + warp * R;
    const unsigned lt = (1u << lane) - 1u;
    for (int d = lane; d < R; d += 32) wc[d] = 0;
    __syncwarp();
    for (int st = 0; st < steps; st++) {
        const int i = i0 + st * 32 + lane;
        const u32 dg = i < n ? (u32)(in[i] >> shift) & (R - 1) : (u32)R;
        const unsigned m = __match_any_sync(0xffffffffu, dg);
        if (dg < (u32)R && !(m & lt)) wc[dg] += __popc(m);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over the warps (in place), digit totals into base
    for (int d = tid; d < R; d += blockDim.x) {
        u32 run = 0;
        for (int w = 0; w < nw; w++) {
            const u32 c = cnt[w * R + d];
            cnt[w * R + d] = run;
            run += c;
        }
        base[d] = run;
    }
    __syncthreads();
    if (warp == 0) {   // exclusive scan of the digit totals: lane l holds digits l * R/32 ..
        constexpr int PER = R / 32 > 0 ? R / 32 : 1;
        u32 loc = 0;
        for (int q = 0; q < PER; q++) loc += lane * PER + q < R ? base[lane * PER + q] : 0u;
        u32 inc = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        u32 run = inc - loc;
        for (int q = 0; q < PER; q++) {
            if (lane * PER + q < R) {
                const u32 c = base[lane * PER + q];
                base[lane * PER + q] = run;
                run += c;
            }
        }
    }
    __syncthreads();
    for (int st = 0; st < steps; st++) {
        const int i = i0 + st * 32 + lane;
        const u64 key = i < n ? in[i] : 0ull;
        const u32 dg = i < n ? (u32)(key >> shift) & (R - 1) : (u32)R;
        const unsigned m = __match_any_sync(0xffffffffu, dg);
        u32 pos = 0;
        if (dg < (u32)R) pos = base[dg] + wc[dg] + __popc(m & lt);
        __syncwarp();
        if (dg < (u32)R) {
            out[pos] = key;
            if (!(m & lt)) wc[dg] += __popc(m);
        }
        __syncwarp();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(CB_THREADS) k_codebook(CompArgs A, CodebookScratch S) {
    if (dev_failed(A.st)) return;
    extern __shared__ __align__(16) u64 cb_dyn[];   // keys[CB_SMEM_KEYS] | weights[2*CB_SMEM_KEYS]
    u64* skeys = cb_dyn;
    __shared__ u32 wcount[33];
    __shared__ u64 lencount[64];
    __shared__ u32 s_lfirst[64], s_llast[64];
    __shared__ u64 firstcode[64];
    __shared__ u32 firstidx[64];
    __shared__ int s_n, s_maxlen, s_np2;
    __shared__ u32 s_rbase[256];
    __shared__ u64 s_total;
    int cap = A.cap;
    int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // 1) alphabet {0} U {s : hist[s] > 0} in symbol order: the bitmap of k_cb_bitmap, then
    //    word-popcount prefixes give every symbol its rank
    // (bitmap and prefixes live in the parent region, which is free before the merge and
    //  after the depth walk; they are rebuilt for the codebook section)
    u32* s_bm = (u32*)(cb_dyn + 3 * CB_SMEM_KEYS);
    u32* s_wpre = s_bm + 2048;
    const int nwords = (cap + 31) >> 5;
    auto build_ranks = [&]() {
        for (int w = tid; w < nwords; w += CB_THREADS) s_bm[w] = S.bm[w];
        __syncthreads();
        const u32 c0 = 2 * tid < nwords ? __popc(s_bm[2 * tid]) : 0u;
        const u32 c1 = 2 * tid + 1 < nwords ? __popc(s_bm[2 * tid + 1]) : 0u;
        u32 inc = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) wcount[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            u32 v = wcount[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            wcount[lane] = v;
            if (lane == 31) s_n = (int)v;
        }
        __syncthreads();
        const u32 ex = (warp ? wcount[warp - 1] : 0u) + inc - (c0 + c1);
        if (2 * tid < nwords) s_wpre[2 * tid] = ex;
        if (2 * tid + 1 < nwords) s_wpre[2 * tid + 1] = ex + c0;
        __syncthreads();
    };
    build_ranks();
    int n = s_n;
    const bool small = n <= CB_SMEM_KEYS;
    // keys and their ping-pong partner: shared memory (the weights region is free until the
    // merge) or global scratch
    u64* keys = small ? skeys : S.keys;
    u64* keys2 = small ? cb_dyn + CB_SMEM_KEYS : S.keys + cap;
    u32 wmax = 0;
    // every alphabet symbol with its rank (= position in symbol order): thread per bitmap word
    auto for_each_symbol = [&](auto f) {
        for (int w = tid; w < nwords; w += CB_THREADS) {
            u32 m = s_bm[w], r = s_wpre[w];
            while (m) {
                const u32 sy = (u32)w * 32u + (u32)(__ffs(m) - 1);
                m &= m - 1u;
                f(r++, sy);
            }
        }
    };
    for_each_symbol([&](u32 i, u32 sy) {
        const u64 w = A.hist[sy];
        keys[i] = (w << 16) | (u64)sy;   // (weight, symbol), in symbol order
        wmax = max(wmax, 64u - (u32)__clzll((long long)w));
    });
    if (tid == 0) s_np2 = 0;
    __syncthreads();
    atomicMax(&s_np2, (int)wmax);
    __syncthreads();
    {
        // stable LSD passes over the weight bytes: (weight, symbol) order.  The digit counters
        // overlay the rank bitmap region (done with above).
        u32* cnt = (u32*)(cb_dyn + 3 * CB_SMEM_KEYS);
        const int wbits = s_np2;
        for (int sh = 0; sh < wbits; sh += 8) {
            cb_radix_pass<8>(keys, keys2, n, 16 + sh, cnt, s_rbase);
            u64* t = keys; keys = keys2; keys2 = t;
        }
        if (small && keys != skeys) {   // the merge's weights go where the keys ended up
            for (int i = tid; i < n; i += CB_THREADS) skeys[i] = keys[i];
            keys2 = keys;
            keys = skeys;
            __syncthreads();
        }
    }
    // 2) two-queue merge (round-synchronous, cb_merge_par; the reference heap with its (weight,
    //    tie) order, encode.py:26-71): node ids: leaves 0..n-1 in sorted order, merged n..2n-2.
    //    Queue heads are kept in registers; weights and parents live in shared memory when the
    //    alphabet fits (u16 parents), else in global scratch.
    u16* par16 = (u16*)(cb_dyn + 3 * CB_SMEM_KEYS);
    const bool w32 = (u64)A.g.nx * (u64)A.g.ny * (u64)A.g.nz < 0xffffffffull;   // total weight fits u32
    {
        u64* W = small ? cb_dyn + CB_SMEM_KEYS : S.w;
        u32* W32 = (u32*)W;
        for (int i = tid; i < n; i += CB_THREADS) {
            if (w32) W32[i] = (u32)(keys[i] >> 16);
            else W[i] = keys[i] >> 16;
        }
        __syncthreads();
    }
    if (tid == 0) s_maxlen = 0;
    if (n == 1) {
        if (tid == 0) {
            if (small) par16[0] = 0xffffu;
            else S.parent[0] = 0xffffffffu;
        }
    } else if (small) {
        auto sp = [&](int i, int mk) { par16[i] = (u16)mk; };
        if (w32) cb_merge_par((u32*)(cb_dyn + CB_SMEM_KEYS), n, sp);
        else cb_merge_par(cb_dyn + CB_SMEM_KEYS, n, sp);
        if (tid == 0) par16[2 * n - 2] = 0xffffu;
    } else {
        auto sp = [&](int i, int mk) { S.parent[i] = (u32)mk; };
        if (w32) cb_merge_par((u32*)S.w, n, sp);
        else cb_merge_par(S.w, n, sp);
        if (tid == 0) S.parent[2 * n - 2] = 0xffffffffu;
    }
    __syncthreads();
    // 3) depths by walking parent pointers (parallel over leaves)
    int root = n == 1 ? 0 : 2 * n - 2;
    int mymax = 0;
    for (int i = tid; i < n; i += CB_THREADS) {
        int d = 0;
        if (n == 1) d = 1;
        else {
            u32 v = (u32)i;
            if (small)
                while (v != (u32)root) { v = par16[v]; d++; }
            else
                while (v != (u32)root) { v = S.parent[v]; d++; }
        }
        u32 sym = (u32)(keys[i] & 0xffff);
        S.lens[sym] = (u8)min(d, 255);
        S.syms[i] = sym;
        mymax = max(mymax, d);
    }
    atomicMax(&s_maxlen, mymax);
    __syncthreads();
    int maxlen = s_maxlen;
    if (maxlen > 57) {
        if (tid == 0) dev_fail(A.st, FTLZ_ERR_INVARIANT, FTLZ_K_CODE_LEN, -1, -1, maxlen, 0, 0);
        return;
    }
    // 4) canonical codes by (length, symbol): one stable counting pass by length over the
    //    symbols in ascending order (ranks rebuilt: the region held the parent pointers)
    __syncthreads();
    build_ranks();
    for_each_symbol([&](u32 i, u32 sym) { keys2[i] = ((u64)S.lens[sym] << 16) | sym; });
    if (tid < 64) { lencount[tid] = 0; s_lfirst[tid] = 0; s_llast[tid] = 0; }
    __syncthreads();
    cb_radix_pass<6>(keys2, keys, n, 16, s_wpre + 2048, s_rbase);
    // keys are sorted by length: each length's count is the span between its boundaries
    for (int i = tid; i < n; i += CB_THREADS) {
        const u32 l = (u32)(keys[i] >> 16);
        if (i == 0 || (u32)(keys[i - 1] >> 16) != l) s_lfirst[l] = (u32)i;
        if (i == n - 1 || (u32)(keys[i + 1] >> 16) != l) s_llast[l] = (u32)(i + 1);
    }
    __syncthreads();
    if (tid < 64) lencount[tid] = (u64)(s_llast[tid] - s_lfirst[tid]);
    __syncthreads();
    if (tid == 0) {
        u64 code = 0;
        u32 idx = 0;
        for (int l = 1; l <= 57; l++) {
            firstcode[l] = code;
            firstidx[l] = idx;
            code = (code + lencount[l]) << 1;
            idx += (u32)lencount[l];
        }
    }
    __shared__ u32 s_symlo, s_symhi;
    if (tid == 0) { s_symlo = 0xffffffffu; s_symhi = 0u; }
    __syncthreads();
    u64 tot = 0;
    u32 slo = 0xffffffffu, shi = 0u;
    for (int i = tid; i < n; i += CB_THREADS) {
        int l = (int)(keys[i] >> 16);
        u32 sym = (u32)(keys[i] & 0xffff);
        u64 code = firstcode[l] + (u64)(i - firstidx[l]);
        A.enc[sym] = (code << 6) | (u64)l;
        tot += (u64)A.hist[sym] * (u64)l;
        if (sym) { slo = min(slo, sym); shi = max(shi, sym); }
    }
    // range of the nonzero symbols (k_enc_pack's window test)
    atomicMin(&s_symlo, slo);
    atomicMax(&s_symhi, shi);
    tot = warp_sum_u64(tot);
    if (tid == 0) s_total = 0;
    __syncthreads();
    if (lane == 0) atomicAdd(&s_total, tot);
    __syncthreads();
    // 5) archive layout (container.py:3-27)
    long long nb = A.g.nb;
    u64 nreg = A.counters[0], nunp = A.layout[LAYOUT_NUNP];
    u64 table_len = 9ull * (u64)nb + 16ull * nreg;
    u64 book_off = 55 + table_len;
    u64 paylen_off = book_off + 4 + 5ull * (u64)n;
    u64 pay_off = paylen_off + 8;
    u64 pay_bytes = (s_total + 7) / 8;
    u64 unp_off = pay_off + pay_bytes;
    u64 sdc_off = unp_off + 4 * nunp;
    u64 total = sdc_off + 16 + (A.store_sum_dc ? 8ull * (u64)nb : 0);
    if (tid == 0) {
        A.layout[LAYOUT_TABLE_LEN] = table_len;
        A.layout[LAYOUT_BOOK_OFF] = book_off;
        A.layout[LAYOUT_NSYM] = (u64)n;
        A.layout[LAYOUT_PAYLEN_OFF] = paylen_off;
        A.layout[LAYOUT_PAY_OFF] = pay_off;
        A.layout[LAYOUT_PAY_BYTES] = pay_bytes;
        A.layout[LAYOUT_UNP_OFF] = unp_off;
        A.layout[LAYOUT_SDC_OFF] = sdc_off;
        A.layout[LAYOUT_TOTAL] = total;
        A.layout[LAYOUT_TOTAL_BITS] = s_total;
        A.layout[LAYOUT_MAXLEN] = (u64)maxlen;
        A.layout[LAYOUT_NREG] = nreg;
        A.layout[LAYOUT_SYMLO] = s_symlo;
        A.layout[LAYOUT_SYMHI] = s_symhi;
        if (total > A.out_cap) dev_fail(A.st, FTLZ_ERR_CAPACITY, 0, -1, -1, (long long)total, 0, 0);
    }
    __syncthreads();
    if (total > A.out_cap) return;
    // 6) codebook section: u32 count, then (u32 symbol, u8 length) in ascending symbol order
    u8* o = A.out + book_off;
    if (tid < 4) o[tid] = (u8)(n >> (8 * tid));
    // symbols in ascending order with their lengths: the input of the length pass (keys2)
    for (int i = tid; i < n; i += CB_THREADS) {
        const u32 sy = (u32)(keys2[i] & 0xffffu);
        u8* e = o + 4 + 5ull * (u64)i;
        e[0] = (u8)sy; e[1] = (u8)(sy >> 8); e[2] = (u8)(sy >> 16); e[3] = (u8)(sy >> 24);
        e[4] = (u8)(keys2[i] >> 16);
    }
}

// ==========================================================================================

// ==========================================================================================
// bins-stage faults (STAGE_BINS_FINALIZED, pipeline.py:468-496).  For every block a fault
// touched, rebuild its 32-bit words (virtual words), run the reference
// verify/correct when protect_bins is on (checksum.py:109-142), and move the histogram
// counts of every word that differs from the clean bin (the reference builds its histogram
// from the verified -- possibly mis-corrected -- bins, pipeline.py:484-492).  The encoder
// then reads these words from fix_scratch.
// warp per block with injected bins faults: verification, correction (checksum.py:109-142,
// candidates tried in increasing j as the reference scans them), histogram fix-up
__global__ void k_fault_bins(CompArgs A, u32* fix_scratch, u8* fixed) {
    if (dev_failed(A.st)) return;
    extern __shared__ u32 fb_smem[];   // vmax words per warp: the block's bin words while verified
    const Geom& g = A.g;
    const int lane = threadIdx.x & 31;
    u32* w = fb_smem + (size_t)(threadIdx.x >> 5) * g.vmax;
    // a warp per block with faults: warp w takes fault w of the block-sorted list when it is its
    // block's first
    const long long nwarp = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long fi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; fi < A.n_faults; fi += nwarp) {
        const long long b = A.faults[fi].block;
        if (fi > 0 && A.faults[fi - 1].block == b) continue;
        const int f0 = (int)fi;
        bool any = false;
        for (int f = f0; f < A.n_faults && A.faults[f].block == b; f++) any |= A.faults[f].target == FTLZ_FAULT_BINS;
        if (!any) continue;
        const BlockInfo B = block_info(g, b);
        const int vol = B.vol;
        u32* wg = fix_scratch + (size_t)b * g.vmax;
        for (int p = lane; p < vol; p += 32) w[p] = A.bins[bins_index(g, b, p)];
        __syncwarp();
        if (lane == 0)
            for (int f = f0; f < A.n_faults && A.faults[f].block == b; f++)
                if (A.faults[f].target == FTLZ_FAULT_BINS) w[A.faults[f].element] ^= 1u << A.faults[f].bit;
        __syncwarp();
        auto sums = [&](u64& s, u64& si) {
            s = 0;
            si = 0;
            for (int p = lane; p < vol; p += 32) { s += w[p]; si += (u64)p * w[p]; }
            s = warp_sum_u64(s);
            si = warp_sum_u64(si);
        };
        if (A.protect_bins) {
            u64 s, si;
            sums(s, si);
            int status = 0;
            if (s != A.bsum[b] || si != A.bisum[b]) {
                status = 2;
                const u64 ds = s - A.bsum[b], dsi = si - A.bisum[b];
                if (ds != 0) {
                    for (int j0 = 0; j0 < vol && status == 2; j0 += 32) {
                        const int j = j0 + lane;
                        const bool cand = j < vol && (u64)j * ds == dsi && (((u64)w[j] - ds) >> 32) == 0;
                        unsigned cm = __ballot_sync(0xffffffffu, cand);
                        while (cm && status == 2) {
                            const int jj = j0 + __ffs(cm) - 1;
                            cm &= cm - 1;
                            const u32 old = w[jj];
                            __syncwarp();
                            if (lane == 0) w[jj] = (u32)((u64)old - ds);
                            __syncwarp();
                            u64 s2, si2;
                            sums(s2, si2);
                            if (s2 == A.bsum[b] && si2 == A.bisum[b]) status = 1;
                            else {
                                __syncwarp();
                                if (lane == 0) w[jj] = old;
                                __syncwarp();
                            }
                        }
                    }
                }
            }
            if (status == 1 && lane == 0) { A.events[b] |= 2; atomicAdd(&A.counters[3], 1u); }
            if (status == 2) {
                if (lane == 0) {
                    A.events[b] |= 8;
                    atomicAdd(&A.counters[3], 1u);
                }
                continue;
            }
        }
        for (int p = lane; p < vol; p += 32) {
            const u32 orig = A.bins[bins_index(g, b, p)];
            if (w[p] == orig) continue;
            if (w[p] >= (u32)A.cap) {
                dev_fail(A.st, FTLZ_ERR_INVARIANT, FTLZ_K_BIN_RANGE, -1, -1, 0, 0, 0);
                continue;
            }
            atomicAdd(&A.hist[orig], ~0ull);   // -1
            atomicAdd(&A.hist[w[p]], 1ull);
        }
        for (int p = lane; p < vol; p += 32) wg[p] = w[p];   // the verified words for k_enc_*
        if (lane == 0) fixed[b] = 1;
    }
}

// ==========================================================================================
// K5: archive assembly (container.py:109-147)
FTLZ_DEV void put_le(u8* o, u64 v, int n) {
    for (int i = 0; i < n; i++) o[i] = (u8)(v >> (8 * i));
}

__global__ void k_assemble(CompArgs A, ftlz_header H) {
    if (dev_failed(A.st)) return;
    const Geom& g = A.g;
    u8* o = A.out;
    long long nb = g.nb;
    long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long stride = (long long)gridDim.x * blockDim.x;
    if (t == 0) {
        o[0] = 'F'; o[1] = 'T'; o[2] = 'L'; o[3] = 'Z'; o[4] = 1; o[5] = 0;
        put_le(o + 6, (u64)H.nx, 8); put_le(o + 14, (u64)H.ny, 8); put_le(o + 22, (u64)H.nz, 8);
        put_le(o + 30, (u64)H.block_edge, 4);
        o[34] = (u8)H.eb_mode;
        put_le(o + 35, A.layout[LAYOUT_EB_BITS], 8);
        put_le(o + 43, (u64)A.cap, 4);
        put_le(o + 47, (u64)nb, 8);
        put_le(o + A.layout[LAYOUT_PAYLEN_OFF], A.layout[LAYOUT_PAY_BYTES], 8);
        u64 so = A.layout[LAYOUT_SDC_OFF];
        u64 raw = A.store_sum_dc ? 8ull * (u64)nb : 0;
        put_le(o + so, raw, 8);
        put_le(o + so + 8, raw, 8);
    }
    u64 unp_off = A.layout[LAYOUT_UNP_OFF], sdc_off = A.layout[LAYOUT_SDC_OFF] + 16;
    for (long long b = t; b < nb; b += stride) {
        u64 ro = 55 + 9ull * (u64)b + 16ull * (u64)A.regpre[b];
        u8 ind = A.ind[b];
        o[ro] = ind;
        ro++;
        if (ind) {
            float4 c = A.coef[b];
            put_le(o + ro, __float_as_uint(c.x), 4);
            put_le(o + ro + 4, __float_as_uint(c.y), 4);
            put_le(o + ro + 8, __float_as_uint(c.z), 4);
            put_le(o + ro + 12, __float_as_uint(c.w), 4);
            ro += 16;
        }
        u32 nu = A.unpc[b];
        put_le(o + ro, nu, 4);
        put_le(o + ro + 4, A.bitlen[b], 4);
        if (nu) {
            const u32* src = A.unp_scratch + (size_t)b * g.vmax;
            u8* d = o + unp_off + 4ull * A.unppre[b];
            for (u32 i = 0; i < nu; i++) put_le(d + 4ull * i, src[i], 4);
        }
        if (A.store_sum_dc) put_le(o + sdc_off + 8ull * (u64)b, A.dcs[b], 8);
    }
}

}  // namespace ftlz
