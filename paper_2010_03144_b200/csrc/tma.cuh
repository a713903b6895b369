// tma.cuh -- per-warp block staging for sm_100a: one cp.async.bulk.tensor (TMA) per block,
// completion on an mbarrier, double-buffered.  Fallback (input rows not 16-byte aligned, so no
// tensor map): per-element cp.async with the same shared-memory layout.
//
// Tile layout (both paths): tile[(i * tye + j) * tz + zs + k] for block-local (i, j, k), where
// zs = (bk * e) mod 4 (the TMA box starts at a 16-byte aligned z: its inner start coordinate must
// be a multiple of 16 bytes, measured on B200 -- others fault) and tz = e + max shift rounded up
// to 4 floats.  Elements outside the block are TMA fill (zeros) or neighbours, never read.
#pragma once
#include <cuda.h>

namespace ftlz {

FTLZ_DEV u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

FTLZ_DEV void mbar_init(u64* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
FTLZ_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
FTLZ_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
FTLZ_DEV void mbar_expect_tx(u64* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
FTLZ_DEV void mbar_wait(u64* bar, u32 parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
FTLZ_DEV void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, u64* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"((u64)map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

struct StageCfg {
    int use_tma;     // tensor map valid
    int tz;          // floats per tile row
    int tye;         // tile rows per i (box extent along y)
    int tile_bytes;  // bytes per tile buffer (TMA box bytes, 128-aligned)
    int box_bytes;   // bytes the TMA transaction delivers
    int pad;
};

// z offset of the block inside its tile row
FTLZ_DEV int zshift(const Geom& g, const BlockInfo& B) { return (int)((B.bk * g.e) & 3); }

// one warp's double-buffered block stager
struct WarpStager {
    unsigned char* base;   // two tiles of `tbytes` (shared memory)
    int tbytes;
    u64* bar;              // 2 mbarriers
    u32 phase;             // bit per buffer

    FTLZ_DEV float* tile(int buf) const { return (float*)(base + buf * tbytes); }

    FTLZ_DEV void init(int lane) {
        phase = 0;
        if (lane == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            mbar_fence_init();
        }
        __syncwarp();
    }

    // issue the copy of block B into buffer `buf` (all lanes call; buffer must be free)
    FTLZ_DEV void issue(const float* __restrict__ x, const Geom& g, const StageCfg& S, const CUtensorMap* map,
                        const BlockInfo& B, int buf, int lane) {
        __syncwarp();
        if (S.use_tma) {
            if (lane == 0) {
                fence_proxy_async();
                mbar_expect_tx(&bar[buf], (u32)S.box_bytes);
                tma_load_3d(tile(buf), map, (int)((B.bk * g.e) & ~3ll), (int)(B.bj * g.e), (int)(B.bi * g.e), &bar[buf]);
            }
        } else {
            long long base = ((B.bi * g.e) * g.ny + B.bj * g.e) * g.nz + B.bk * g.e;
            int byz = B.by * B.bz;
            for (int p = lane; p < B.vol; p += 32) {
                int i = p / byz, rem = p - i * byz, j = rem / B.bz, k = rem - j * B.bz;
                unsigned sa = smem_u32(tile(buf) + (i * S.tye + j) * S.tz + zshift(g, B) + k);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa),
                             "l"(x + base + ((long long)i * g.ny + j) * g.nz + k));
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    }
    // wait for buffer `buf`; `more` = another copy was issued after it (cp.async group count)
    FTLZ_DEV void wait(const StageCfg& S, int buf, bool more) {
        if (S.use_tma) {
            mbar_wait(&bar[buf], (phase >> buf) & 1u);
            phase ^= 1u << buf;
        } else {
            if (more) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
    }
};

}  // namespace ftlz
