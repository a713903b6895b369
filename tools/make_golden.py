"""Generate tests/golden/ by running the reference `ftlz` package (Python) in this container.

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py [--large]

The reference cannot travel to the GPU box, so its outputs are committed as fixtures:
  tests/golden/<case>.npz   input field, archive bytes, decompressed output (small cases)
  tests/golden/manifest.json  per case: request, config, faults, expected reports/errors,
                              SHA-256 of input / archive / output (all cases)
`--large` adds the BASELINE configs c1..c5 at full size (hash-only; c3 takes minutes).

Faults are applied through the reference's own hook seam with the semantics of
faults.py:157-189 (one XOR per (block, element, bit); decomp hook armed once=True).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import ftlz  # noqa: E402
from ftlz import hooks  # noqa: E402
from ftlz.errors import FtlzError  # noqa: E402

from tools import synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def sha(buf) -> str:
    return hashlib.sha256(memoryview(np.ascontiguousarray(buf)).cast("B")).hexdigest()


def cfg_obj(cfg: dict):
    base = dict(protect_input=True, protect_bins=True, duplicate_eval=True, store_sum_dc=True,
                block_edge=10)
    base.update(cfg)
    cap = base.pop("bin_capacity", None)
    if cap is not None:
        base["quant"] = ftlz.QuantConfig(cap)
    return ftlz.FtConfig(**base)


def run_compress(values, mode, value, cfg, faults, override):
    field = ftlz.Field.from_array(values)
    eb = ftlz.ErrorBound(mode, value)
    armed = []
    byt = {}
    for t, b, e, bit in faults:
        byt.setdefault(t, []).append((b, e, bit))

    def h_input(working, grid):
        for b, e, bit in byt["input"]:
            i, j, k = grid.cell_of_block(b, e)
            working[i, j, k: k + 1].view(np.uint32)[0] ^= np.uint32(1 << bit)

    def h_bins(bins_list, grid):
        for b, e, bit in byt["bins"]:
            bins_list[b][e] ^= np.uint32(1 << bit)

    def h_coef(coeffs_all, grid):
        for b, e, bit in byt["regression"]:
            coeffs_all[b: b + 1].view(np.uint32)[0, e] ^= np.uint32(1 << bit)

    def h_est(est_reg, est_lor):
        for b, e, bit in byt["sampling"]:
            arr = est_reg if e == 0 else est_lor
            arr[b: b + 1].view(np.uint64)[0] ^= np.uint64(1 << bit)

    dups = [(t, b, e, bit // 64 + 1, bit % 64) for t, b, e, bit in faults if t.startswith("dup_")]

    def h_dup(tag, rnd, arr):
        # STAGE_DUP_EVAL fires inside duplicated_eval with the whole batch of one (extent group,
        # predictor) subset: (n, bx, by, bz) for regression, (n, m) per Lorenzo wavefront.  The
        # calling _compress_rows frame names the batch's blocks and the current wavefront.
        fr = sys._getframe(1)
        while fr is not None and fr.f_code.co_name != "_compress_rows":
            fr = fr.f_back
        loc = fr.f_locals
        blocks = loc["ids"][loc["rows"]]
        out = None
        for t, b, e, r, bit in dups:
            if r != rnd or t != "dup_" + tag:
                continue
            hit = np.flatnonzero(blocks == b)
            if not hit.size:
                continue
            if arr.ndim == 4:
                q = e
            else:
                _, by, bz = loc["extent"]
                li, rem = divmod(e, by * bz)
                lj, lk = divmod(rem, bz)
                qq = np.flatnonzero((loc["ii"] == li) & (loc["jj"] == lj) & (loc["kk"] == lk))
                if not qq.size:
                    continue
                q = int(qq[0])
            if out is None:
                out = np.array(arr, dtype=np.float64, copy=True)
            v = out.reshape(len(blocks), -1)
            v[hit[0]: hit[0] + 1, q: q + 1].view(np.uint64)[0, 0] ^= np.uint64(1 << bit)
        return arr if out is None else out

    if dups:
        hooks.arm(hooks.STAGE_DUP_EVAL, h_dup)
    if "input" in byt:
        hooks.arm(hooks.STAGE_INPUT_AFTER_CHECKSUM, h_input)
    if "bins" in byt:
        hooks.arm(hooks.STAGE_BINS_FINALIZED, h_bins)
    if "regression" in byt:
        hooks.arm(hooks.STAGE_COEFFS_FITTED, h_coef)
    if "sampling" in byt:
        hooks.arm(hooks.STAGE_ESTIMATES, h_est)
    try:
        ov = None
        if override:
            ov = {int(b): ftlz.PredictorKind(int(k)) for b, k in override.items()}
        stream, rep = ftlz.compress(field, eb, cfg_obj(cfg), predictor_override=ov)
        return ftlz.serialize(stream), rep.to_dict(), None
    except FtlzError as exc:
        return None, None, {"cls": type(exc).__name__, "msg": str(exc)}
    finally:
        hooks.disarm_all()
        del armed


def run_decompress(data, faults):
    dec = [(b, e, bit) for t, b, e, bit in faults if t == "decomp"]
    try:
        stream = ftlz.parse(data)
    except FtlzError as exc:
        return None, None, {"cls": type(exc).__name__, "msg": str(exc)}

    def h_dec(out, grid):
        for b, e, bit in dec:
            i, j, k = grid.cell_of_block(b, e)
            out[i, j, k: k + 1].view(np.uint32)[0] ^= np.uint32(1 << bit)

    if dec:
        hooks.arm(hooks.STAGE_DECOMP_BEFORE_VERIFY, h_dec, once=True)
    try:
        out, rep = ftlz.decompress(stream)
    finally:
        hooks.disarm_all()
    return (None if out is None else np.array(out.values)), rep.to_dict(), None


def small_cases():
    S = ftlz.synth_field
    cases = []

    def add(name, values, mode, value, cfg=None, faults=(), override=None, extra=None):
        # keep every fault inside its block (faults.py:_pick draws element < volume)
        vols = synth.block_volumes(np.shape(values), (cfg or {}).get("block_edge", 10))
        faults = [(t, b, e % (4 if t == "regression" else 2 if t == "sampling" else int(vols[b])),
                   bit) for t, b, e, bit in faults]
        cases.append(dict(name=name, values=np.ascontiguousarray(values, np.float32), mode=mode,
                          value=value, cfg=cfg or {}, faults=list(faults), override=override,
                          extra=extra or {}))

    A, R = "absolute", "value_range_relative"
    # test_pipeline.py:78-104 awkward dims with edge 5
    for kind, ebv in (("mixed", 1e-3), ("noise", 1e-4), ("sine", 1e-2)):
        add(f"pipe_{kind}_13x11x10_e5", S(kind, (13, 11, 10), seed=31).values, A, ebv,
            {"block_edge": 5})
    add("payload_14x10x9_e4", S("mixed", (14, 10, 9), seed=8).values, A, 1e-3, {"block_edge": 4})
    add("constant_40", S("constant", (40, 40, 40), seed=1).values, A, 1e-3)
    add("degenerate_rel_constant", S("constant", (12, 12, 12), seed=1).values, R, 1e-3)
    add("flat2d_1x32x24", S("mixed", (1, 32, 24), seed=19).values, A, 1e-3)
    add("relative_sine_16", S("sine", (16, 16, 16), seed=9).values, R, 1e-3)
    add("transparency_on_24x20x22", S("mixed", (24, 20, 22), seed=3).values, A, 1e-2)
    add("transparency_off_24x20x22", S("mixed", (24, 20, 22), seed=3).values, A, 1e-2,
        {"protect_input": False, "protect_bins": False, "duplicate_eval": False,
         "store_sum_dc": False})
    add("noise_16_e8_1e-4", S("noise", (16, 16, 16), seed=7).values, A, 1e-4, {"block_edge": 8})
    add("noise_20_1e-6_bigalphabet", S("noise", (20, 20, 20), seed=5).values, A, 1e-6)
    add("mixed_12x9x7_e4_unprot", S("mixed", (12, 9, 7), seed=21).values, A, 1e-3,
        {"block_edge": 4, "protect_input": False, "protect_bins": False,
         "duplicate_eval": False, "store_sum_dc": False})
    add("sine_20_e2", S("sine", (20, 20, 20), seed=2).values, A, 1e-3, {"block_edge": 2})
    add("mixed_33x17x70_e16", S("mixed", (33, 17, 70), seed=4).values, R, 1e-4, {"block_edge": 16})
    add("mixed_20x20x20_e64", S("mixed", (20, 20, 20), seed=4).values, A, 1e-3, {"block_edge": 64})
    add("cap_256_noise", S("noise", (16, 16, 16), seed=3).values, A, 1e-2, {"bin_capacity": 256})
    # lognormal with wide dynamic range (regression-heavy, like c3) at reduced size
    g = synth.grf((32, 32, 48), 2.5, 11)
    add("lognormal_32x32x48", np.exp(g), R, 1e-3)
    add("grf2d_1x90x180", (synth.grf((90, 180), 3.0, 4, std=5.0) + 250.0).reshape(1, 90, 180), R, 1e-4)
    # special values (absolute bound): NaN / inf / -0.0 / huge / subnormal
    rng = np.random.default_rng(77)
    sp = rng.standard_normal((15, 14, 13)).astype(np.float32)
    sp[0, 0, :] = -0.0
    sp[:10, :10, :10][3, 3, 3] = np.nan
    sp[11, 2, 7] = np.inf
    sp[12, 5, 1] = -np.inf
    sp[4, 13, 12] = 3.0e38
    sp[5, 5, 5] = 1e-42
    sp[10:, 10:, 10:] = -0.0   # an all-negative-zero block
    add("special_values_abs", sp, A, 1e-3)
    add("special_values_rel", sp, R, 1e-3)
    # fault injection through the hook seam (faults.py:157-189)
    base = S("mixed", (16, 14, 12), seed=2).values
    fa = [("input", 3, 17, 30), ("input", 7, 0, 5), ("input", 20, 99, 31)]
    add("fault_input_protected", base, A, 1e-3, {"block_edge": 5}, fa)
    add("fault_input_unprotected", base, A, 1e-3, {"block_edge": 5, "protect_input": False}, fa)
    fb = [("bins", 1, 4, 3), ("bins", 9, 60, 17), ("bins", 22, 0, 31)]
    add("fault_bins_protected", base, A, 1e-3, {"block_edge": 5}, fb)
    add("fault_bins_unprotected_range", base, A, 1e-3, {"block_edge": 5, "protect_bins": False}, fb)
    add("fault_bins_unprotected_low", base, A, 1e-3, {"block_edge": 5, "protect_bins": False},
        [("bins", 4, 10, 1), ("bins", 11, 3, 0)])
    add("fault_bins_double_uncorrectable", base, A, 1e-3, {"block_edge": 5},
        [("bins", 6, 2, 1), ("bins", 6, 9, 4)])
    add("fault_input_double_uncorrectable", base, A, 1e-3, {"block_edge": 5},
        [("input", 8, 2, 1), ("input", 8, 9, 4), ("input", 2, 5, 6), ("input", 2, 6, 6)])
    add("fault_coeff", base, A, 1e-3, {"block_edge": 5},
        [("regression", 0, 0, 30), ("regression", 5, 1, 22), ("regression", 13, 3, 2)])
    add("fault_estimate", base, A, 1e-3, {"block_edge": 5},
        [("sampling", 2, 0, 62), ("sampling", 4, 1, 63), ("sampling", 17, 0, 10)])
    add("fault_decomp_protected", base, A, 1e-3, {"block_edge": 5},
        [("decomp", 3, 10, 22), ("decomp", 12, 0, 31), ("decomp", 30, 124, 0)])
    add("fault_decomp_unprotected", base, A, 1e-3,
        {"block_edge": 5, "protect_input": False, "protect_bins": False,
         "duplicate_eval": False, "store_sum_dc": False},
        [("decomp", 3, 10, 30)])
    # duplicated evaluation (STAGE_DUP_EVAL, pipeline.py:157-179): bit = 64 * (round - 1) + b.
    # Regression blocks of `base` (edge 5): 4, 6, 8, 15, 17, 26-31, 34; the rest are Lorenzo.
    R1, R2, R3 = 0, 64, 128
    add("dup_majority", base, A, 1e-3, {"block_edge": 5},
        [("dup_reconstruct", 4, 7, R1 + 52), ("dup_predict", 4, 20, R2 + 40),
         ("dup_predict", 0, 3, R1 + 45), ("dup_reconstruct", 2, 30, R2 + 10),
         ("dup_predict", 30, 11, R1 + 63), ("dup_reconstruct", 8, 6, R1 + 62)])
    add("dup_triple_disagreement", base, A, 1e-3, {"block_edge": 5},
        [("dup_reconstruct", 4, 7, R1 + 51), ("dup_reconstruct", 4, 7, R3 + 30),
         ("dup_predict", 0, 12, R1 + 45), ("dup_predict", 0, 12, R2 + 20),
         ("dup_predict", 15, 40, R1 + 33), ("dup_predict", 15, 40, R2 + 34), ("dup_predict", 15, 40, R3 + 35),
         ("dup_reconstruct", 5, 0, R1 + 1), ("dup_reconstruct", 5, 0, R3 + 2)])
    add("dup_same_flip_rounds_1_2", base, A, 1e-3, {"block_edge": 5},
        [("dup_predict", 6, 9, R1 + 48), ("dup_predict", 6, 9, R2 + 48),
         ("dup_reconstruct", 3, 14, R1 + 40), ("dup_reconstruct", 3, 14, R2 + 40)])
    add("dup_round3_only", base, A, 1e-3, {"block_edge": 5},
        [("dup_predict", 4, 5, R3 + 60), ("dup_reconstruct", 1, 9, R3 + 61)])
    add("dup_unprotected", base, A, 1e-3, {"block_edge": 5, "duplicate_eval": False},
        [("dup_predict", 4, 3, R1 + 50), ("dup_reconstruct", 1, 4, R1 + 33), ("dup_predict", 6, 2, R2 + 50),
         ("dup_predict", 7, 8, R1 + 45)])
    dplan = synth.fault_plan(len(synth.block_volumes((30, 30, 30), 10)), synth.block_volumes((30, 30, 30), 10),
                             seed=99, frac=0.3)
    add("dup_plan_30", S("mixed", (30, 30, 30), seed=5).values, R, 1e-3, {},
        [("dup_predict" if t % 2 else "dup_reconstruct", b, e, (t % 2) * 64 + 20 + t) for b, e, t in dplan])
    add("override_mix", S("mixed", (20, 15, 10), seed=14).values, A, 1e-3, {"block_edge": 5},
        override={0: 1, 3: 0, 7: 1, 11: 0, 23: 1})
    # c5-style plan at reduced size: 10% of blocks, bits 0..31, three targets
    c5v = S("mixed", (30, 30, 30), seed=5).values
    vols = synth.block_volumes((30, 30, 30), 10)
    plan = synth.fault_plan(len(vols), vols, seed=12345, frac=0.1)
    for tgt in ("input", "bins", "decomp"):
        add(f"c5mini_{tgt}", c5v, R, 1e-3, {}, [(tgt, b, e, t) for b, e, t in plan])
    # the full c1 config (64^3, relative 1e-3)
    add("c1", synth.c1(), R, 1e-3)
    return cases


def corrupt_cases(archive: bytes):
    """(name, bytes) variants of a valid archive for parse/decompress error parity."""
    out = []
    n = len(archive)
    cuts = sorted(set([0, 1, 4, 30, 54, 55, 56, 60, 100, n // 3, n // 2, n - 30, n - 17, n - 16,
                       n - 9, n - 8, n - 1]))
    for c in cuts:
        if 0 <= c < n:
            out.append((f"cut_{c}", archive[:c]))
    out.append(("trailing", archive + b"\x00"))
    b = bytearray(archive); b[0:4] = b"XTLZ"; out.append(("magic", bytes(b)))
    b = bytearray(archive); b[4] = 99; out.append(("version", bytes(b)))
    b = bytearray(archive); b[6:14] = (0).to_bytes(8, "little"); out.append(("dims", bytes(b)))
    b = bytearray(archive); b[30:34] = (1).to_bytes(4, "little"); out.append(("edge", bytes(b)))
    b = bytearray(archive); b[34] = 7; out.append(("mode", bytes(b)))
    b = bytearray(archive); b[35:43] = np.float64(-1.0).tobytes(); out.append(("eb", bytes(b)))
    b = bytearray(archive); b[35:43] = np.float64(np.inf).tobytes(); out.append(("eb_inf", bytes(b)))
    b = bytearray(archive); b[43:47] = (1000).to_bytes(4, "little"); out.append(("cap", bytes(b)))
    b = bytearray(archive); b[47:55] = (999).to_bytes(8, "little"); out.append(("count", bytes(b)))
    b = bytearray(archive); b[55] = 2; out.append(("indicator0", bytes(b)))
    b = bytearray(archive); b[5] = 9; out.append(("codec", bytes(b)))
    return out


def payload_flip_cases(archive: bytes, stream):
    table = sum(9 + (16 if r.predictor == 1 else 0) for r in stream.records)
    book = 4 + 5 * len(stream.code_lengths)
    off = 55 + table + book + 8
    plen = len(stream.payload)
    res = []
    for pos in sorted(set(np.linspace(0, plen - 1, 12).astype(int).tolist())):
        b = bytearray(archive)
        b[off + pos] ^= 0xFF
        res.append((f"payflip_{pos}", bytes(b)))
    # codebook damage: swap first two symbols, bad length, kraft
    boff = 55 + table
    b = bytearray(archive); b[boff + 4: boff + 8] = (70000).to_bytes(4, "little")
    res.append(("book_symrange", bytes(b)))
    b = bytearray(archive); b[boff + 8] = 0
    res.append(("book_len0", bytes(b)))
    b = bytearray(archive); b[boff + 8] = 60
    res.append(("book_len60", bytes(b)))
    b = bytearray(archive)
    for t in range(min(4, len(stream.code_lengths))):
        b[boff + 4 + 5 * t + 4] = 1
    res.append(("book_kraft", bytes(b)))
    b = bytearray(archive); b[boff + 4 + 5: boff + 4 + 9] = (0).to_bytes(4, "little")
    res.append(("book_order", bytes(b)))
    # sum_dc section lengths
    b = bytearray(archive); b[-8 * len(stream.records) - 16] ^= 1
    res.append(("sumdc_rawlen", bytes(b)))
    b = bytearray(archive); b[-8 * len(stream.records) - 8] ^= 1
    res.append(("sumdc_storedlen", bytes(b)))
    # sum_dc value flip -> re-execution cannot fix -> terminal SDC at that block
    b = bytearray(archive); b[-8 * 3] ^= 0x10
    res.append(("sumdc_value", bytes(b)))
    # record bit_length/unpred_count tampering
    b = bytearray(archive); b[55 + 1 + (16 if stream.records[0].predictor else 0)] ^= 1
    res.append(("rec0_unpred", bytes(b)))
    b = bytearray(archive); b[55 + 5 + (16 if stream.records[0].predictor else 0)] ^= 1
    res.append(("rec0_bitlen", bytes(b)))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    ap.add_argument("--only", default=None)
    ap.add_argument("--region", action="store_true", help="region-extraction fixtures only")
    ap.add_argument("--campaign", action="store_true", help="fault-campaign fixtures only")
    ap.add_argument("--codec", action="store_true", help="backend codec 1 (run-length) fixtures only")
    ap.add_argument("--truncation", action="store_true", help="every-byte truncation sweep only")
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    mpath = os.path.join(OUT, "manifest.json")
    manifest = json.load(open(mpath)) if os.path.exists(mpath) else {"cases": {}, "corrupt": {}, "large": {}}
    manifest["generator"] = {"numpy": np.__version__, "ftlz": ftlz.__version__,
                             "script": "tools/make_golden.py"}
    if args.truncation:
        # test_container.py:59-63: every proper prefix of an archive fails parse with CorruptStream;
        # the class and message (with its offset) of each cut, for three small archives
        res = {}
        for src in ("pipe_sine_13x11x10_e5", "relative_sine_16", "mixed_12x9x7_e4_unprot"):
            arch = np.load(os.path.join(OUT, src + ".npz"))["archive"].tobytes()
            errs = []
            for cut in range(len(arch)):
                try:
                    ftlz.parse(arch[:cut])
                    errs.append(None)
                except FtlzError as exc:
                    errs.append([type(exc).__name__, str(exc)])
            msgs = sorted({tuple(e) for e in errs if e})
            pos = {m: i for i, m in enumerate(msgs)}
            res[src] = {"len": len(arch), "messages": [list(m) for m in msgs],
                        "index": [-1 if e is None else pos[tuple(e)] for e in errs]}
        json.dump(res, open(os.path.join(OUT, "truncation.json"), "w"), separators=(",", ":"))
        print("truncation", {k: v["len"] for k, v in res.items()})
        return
    if args.codec:
        # backend codec 1 (encode.py:287-312) through serialize/parse (container.py:134-145,241-262)
        from ftlz import encode as ENC

        rng = np.random.default_rng(123)
        vecs = {"empty": b"", "one": b"\x07", "run255": b"\x00" * 255, "run256": b"\x00" * 256,
                "run510": b"\xab" * 510, "run1000": b"\x01" * 1000,
                "mixed": bytes(rng.integers(0, 3, 5000, dtype=np.uint8)),
                "random": bytes(rng.integers(0, 256, 20000, dtype=np.uint8)),
                "blocks": b"".join(bytes([v]) * int(n) for v, n in zip(rng.integers(0, 256, 300),
                                                                      rng.integers(1, 700, 300)))}
        arrs = {}
        for k, v in vecs.items():
            arrs[f"in_{k}"] = np.frombuffer(v, np.uint8)
            arrs[f"out_{k}"] = np.frombuffer(ENC.backend_apply(v, 1), np.uint8)
        np.savez_compressed(os.path.join(OUT, "rle_vectors.npz"), **arrs)
        cases = {}
        S = ftlz.synth_field
        A, R = "absolute", "value_range_relative"
        specs = [("c1_constant_30", S("constant", (30, 30, 30), seed=1).values, A, 1e-3, {}),
                 ("c1_mixed_24x20x22", S("mixed", (24, 20, 22), seed=3).values, A, 1e-2, {}),
                 ("c1_noise_20_1e-6", S("noise", (20, 20, 20), seed=5).values, A, 1e-6, {}),
                 ("c1_lognormal_32x32x48", np.exp(synth.grf((32, 32, 48), 2.5, 11)), R, 1e-3, {}),
                 ("c1_unprot_13x11x10_e5", S("mixed", (13, 11, 10), seed=31).values, A, 1e-3,
                  {"block_edge": 5, "protect_input": False, "protect_bins": False,
                   "duplicate_eval": False, "store_sum_dc": False})]
        for name, vals, mode, ebv, cfg in specs:
            vals = np.ascontiguousarray(vals, np.float32)
            cfg = dict(cfg, codec_id=1)
            arch, crep, err = run_compress(vals, mode, ebv, cfg, [], None)
            assert err is None, err
            out, drep, derr = run_decompress(arch, [])
            stream = ftlz.parse(arch)
            # corrupt variants of the run-length sections
            nb = len(stream.records)
            table = sum(9 + (16 if r.predictor == 1 else 0) for r in stream.records)
            poff = 55 + table + 4 + 5 * len(stream.code_lengths)      # u64 stored payload length
            plen = int.from_bytes(arch[poff:poff + 8], "little")
            corrupt = {}
            b = bytearray(arch); b[poff:poff + 8] = (plen - 1).to_bytes(8, "little"); del b[poff + 8 + plen - 1]
            corrupt["pay_odd"] = bytes(b)
            b = bytearray(arch); b[poff + 8] = 0
            corrupt["pay_zero"] = bytes(b)
            b = bytearray(arch); b[poff:poff + 8] = (plen - 2).to_bytes(8, "little"); del b[poff + 8 + plen - 2:poff + 8 + plen]
            corrupt["pay_short"] = bytes(b)
            b = bytearray(arch); b[poff + 8] = 255
            corrupt["pay_longrun"] = bytes(b)
            if cfg.get("store_sum_dc", True):
                soff = poff + 8 + plen + len(stream.unpred_words)   # (raw, stored) lengths
                slen = int.from_bytes(arch[soff + 8:soff + 16], "little")
                b = bytearray(arch); b[soff + 8:soff + 16] = (slen - 1).to_bytes(8, "little"); del b[soff + 16 + slen - 1]
                corrupt["sdc_odd"] = bytes(b)
                b = bytearray(arch); b[soff + 16] = 0
                corrupt["sdc_zero"] = bytes(b)
                b = bytearray(arch); b[soff + 16] = min(255, b[soff + 16] + 1)
                corrupt["sdc_long"] = bytes(b)
            cres = {}
            for k, blob in corrupt.items():
                o2, r2, e2 = run_decompress(blob, [])
                cres[k] = {"error": e2, "report": r2, "output_sha256": None if o2 is None else sha(o2),
                           "len": len(blob)}
            np.savez_compressed(os.path.join(OUT, f"{name}.npz"), input=vals,
                                archive=np.frombuffer(arch, np.uint8),
                                output=np.zeros(0, np.float32) if out is None else out,
                                **{f"corrupt_{k}": np.frombuffer(v, np.uint8) for k, v in corrupt.items()})
            cases[name] = {"mode": mode, "value": ebv, "cfg": cfg, "archive_sha256": sha(np.frombuffer(arch, np.uint8)),
                           "archive_len": len(arch), "output_sha256": None if out is None else sha(out),
                           "compress_report": crep, "decompress_report": drep, "corrupt": cres}
        manifest["codec1"] = cases
        json.dump(manifest, open(mpath, "w"), indent=1, sort_keys=True)
        print("codec1", list(cases))
        return
    if args.campaign:
        # faults.run_trial / run_campaign (faults.py:143-367): every target, both protections
        from ftlz import faults as FT

        f = ftlz.synth_field("mixed", (16, 14, 12), seed=21)
        np.savez_compressed(os.path.join(OUT, "campaign.npz"), input=f.values)
        ebs = [ftlz.ErrorBound.absolute(1e-3), ftlz.ErrorBound.relative(1e-3)]
        cfgs = {"protected": ftlz.FtConfig.protected(block_edge=5),
                "unprotected": ftlz.FtConfig.unprotected(block_edge=5)}
        seed, trials = 7, 4
        rep = FT.run_campaign(f, ebs, cfgs, trials=trials, seed=seed, targets=FT.TARGETS, field_note="golden")
        outcomes = []
        ci = 0
        for cname, cfg in cfgs.items():
            for tgt in FT.TARGETS:
                for eb in ebs:
                    ref = FT.fault_free_reference(f, eb, cfg)
                    for t in range(trials):
                        plan = FT.InjectionPlan(target=tgt, seed=FT.trial_seed(seed, ci, t))
                        o = FT.run_trial(f, eb, cfg, plan, ref)
                        outcomes.append({"cfg": cname, "target": tgt, "eb": [eb.mode, eb.value], "trial": t,
                                         "classification": o.classification, "corrected": o.corrected,
                                         "max_abs_error": o.max_abs_error, "ratio": o.ratio,
                                         "bit_identical_output": o.bit_identical_output,
                                         "bit_identical_archive": o.bit_identical_archive,
                                         "compress_events": o.compress_events,
                                         "decompress_events": o.decompress_events, "detail": o.detail})
                    ci += 1
        manifest["campaign"] = {"seed": seed, "trials": trials, "rows": rep.rows(), "outcomes": outcomes,
                                "input_sha256": sha(f.values)}
        json.dump(manifest, open(mpath, "w"), indent=1, sort_keys=True)
        print("campaign", len(outcomes))
        return
    if args.region:
        # decompress_region (pipeline.py:726-795) on clean and payload-damaged archives
        res = {}
        for src in ("payload_14x10x9_e4", "pipe_noise_13x11x10_e5", "mixed_33x17x70_e16"):
            z = np.load(os.path.join(OUT, src + ".npz"))
            arch = z["archive"].tobytes()
            blobs = [("clean", arch)]
            if src != "mixed_33x17x70_e16":
                cz = np.load(os.path.join(OUT, f"corrupt_{src}.npz"))
                blobs += [(k, cz[k].tobytes()) for k in sorted(cz.files) if k.startswith("payflip_")]
            dims = ftlz.parse(arch).dims
            regions = [((0, 0, 0), tuple(dims)),
                       ((1, 2, 3), tuple(max(4, d - 2) for d in dims)),
                       ((0, 0, 0), (min(5, dims[0]), min(4, dims[1]), min(3, dims[2]))),
                       ((dims[0] - 1, dims[1] - 1, dims[2] - 1), tuple(dims))]
            for bname, blob in blobs:
                stream = ftlz.parse(blob)
                for ri, reg in enumerate(regions):
                    out, rep = ftlz.decompress_region(stream, reg)
                    key = f"{src}|{bname}|{ri}"
                    res[key] = {"region": [list(reg[0]), list(reg[1])], "status": rep.status,
                                "detail": rep.detail, "reexecuted": list(rep.decomp_block_reexecuted),
                                "output_sha256": None if out is None else sha(out.values)}
        manifest["region"] = res
        json.dump(manifest, open(mpath, "w"), indent=1, sort_keys=True)
        print("region", len(res))
        return
    if not args.large:
        for c in small_cases():
            if args.only and args.only not in c["name"]:
                continue
            t0 = time.time()
            data, crep, cerr = run_compress(c["values"], c["mode"], c["value"], c["cfg"],
                                            c["faults"], c["override"])
            entry = {k: c[k] for k in ("mode", "value", "cfg", "faults")}
            entry["override"] = {str(k): v for k, v in (c["override"] or {}).items()}
            entry["dims"] = list(c["values"].shape)
            entry["input_sha256"] = sha(c["values"])
            arrays = {"input": c["values"]}
            if cerr:
                entry["compress_error"] = cerr
            else:
                entry["archive_sha256"] = sha(np.frombuffer(data, np.uint8))
                entry["archive_len"] = len(data)
                entry["compress_report"] = crep
                arrays["archive"] = np.frombuffer(data, np.uint8)
                out, drep, derr = run_decompress(data, c["faults"])
                entry["decompress_report"] = drep
                if out is not None:
                    entry["output_sha256"] = sha(out)
                    arrays["output"] = out
            np.savez_compressed(os.path.join(OUT, c["name"] + ".npz"), **arrays)
            manifest["cases"][c["name"]] = entry
            print(c["name"], f"{time.time() - t0:.2f}s", entry.get("archive_len"), cerr or "")
        # parse / decompress error parity on two archives (protected + unprotected)
        for src in ("payload_14x10x9_e4", "pipe_noise_13x11x10_e5", "mixed_12x9x7_e4_unprot"):
            z = np.load(os.path.join(OUT, src + ".npz"))
            arch = z["archive"].tobytes()
            stream = ftlz.parse(arch)
            variants = corrupt_cases(arch) + payload_flip_cases(arch, stream)
            res = {}
            blobs = {}
            for name, blob in variants:
                out, drep, derr = run_decompress(blob, [])
                r = {"len": len(blob), "sha256": sha(np.frombuffer(blob, np.uint8))}
                if derr:
                    r["error"] = derr
                else:
                    r["decompress_report"] = drep
                    r["output_sha256"] = None if out is None else sha(out)
                res[name] = r
                blobs[name] = np.frombuffer(blob, np.uint8)
            manifest["corrupt"][src] = res
            np.savez_compressed(os.path.join(OUT, f"corrupt_{src}.npz"), **blobs)
            print("corrupt", src, len(res))
    else:
        for name in ("c1", "c4", "c2", "c2_1e-4", "c3", "c5"):
            if args.only and args.only != name:
                continue
            t0 = time.time()
            f = synth.field(name)
            mode, v = synth.CONFIGS[name]["eb"]
            entry = {"dims": list(f.shape), "mode": mode, "value": v, "input_sha256": sha(f)}
            if name == "c5":
                vols = synth.block_volumes(f.shape, 10)
                plan = synth.fault_plan(len(vols), vols)
                entry["plan_sha256"] = hashlib.sha256(json.dumps(plan).encode()).hexdigest()
                entry["n_faults"] = len(plan)
                for tgt in ("input", "bins", "decomp"):
                    fl = [(tgt, b, e, t) for b, e, t in plan]
                    data, crep, cerr = run_compress(f, mode, v, {}, fl, None)
                    out, drep, _ = run_decompress(data, fl)
                    entry[tgt] = {"archive_sha256": sha(np.frombuffer(data, np.uint8)),
                                  "archive_len": len(data),
                                  "n_input_corrected": len(crep["input_corrected"]),
                                  "n_bins_corrected": len(crep["bins_corrected"]),
                                  "input_corrected_sha256": hashlib.sha256(json.dumps(crep["input_corrected"]).encode()).hexdigest(),
                                  "bins_corrected_sha256": hashlib.sha256(json.dumps(crep["bins_corrected"]).encode()).hexdigest(),
                                  "n_reexecuted": len(drep["decomp_block_reexecuted"]),
                                  "reexecuted_sha256": hashlib.sha256(json.dumps(drep["decomp_block_reexecuted"]).encode()).hexdigest(),
                                  "status_c": crep["status"], "status_d": drep["status"],
                                  "output_sha256": None if out is None else sha(out)}
                    print(name, tgt, entry[tgt], flush=True)
            else:
                data, crep, cerr = run_compress(f, mode, v, {}, [], None)
                out, drep, _ = run_decompress(data, [])
                entry.update({"archive_sha256": sha(np.frombuffer(data, np.uint8)),
                              "archive_len": len(data), "compress_report": crep,
                              "decompress_report": drep, "output_sha256": sha(out)})
            entry["seconds"] = round(time.time() - t0, 1)
            manifest["large"][name] = entry
            json.dump(manifest, open(mpath, "w"), indent=1, sort_keys=True)
            print(name, entry.get("archive_len"), entry["seconds"], flush=True)
    json.dump(manifest, open(mpath, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
