"""Golden fixtures for byte-view keys and n-grams, made by the UNMODIFIED
reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_bytes.py

Writes ``golden_bytes.npz``: content-hash known answers (hashing.py:56-66 and
BytePrefixHasher.hash_views :98-106), ``build_ngrams`` outputs for a few texts
(ngrams.py:23-89), semisort outputs of n-gram records in both modes with
telemetry (core.py:566-598 with BytesKeyAdapter, adapters.py:200-275), and
histogram / collect_reduce(summing64) pairs of n-gram records with telemetry
(aggregate.py:267-299).  The texts are generated here from a seeded
vocabulary; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

import semisort as S  # noqa: E402
from semisort.hashing import BytePrefixHasher, hash_bytes  # noqa: E402
from semisort.ngrams import build_ngrams, ngram_adapter  # noqa: E402


def synth_text(seed: int, words: int, vocab: int) -> bytes:
    """Space/punctuation separated words from a seeded vocabulary, Zipf-ish use."""
    r = np.random.default_rng(seed)
    lens = r.integers(1, 11, vocab)
    letters = np.frombuffer(b"abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ", dtype=np.uint8)
    voc = [bytes(letters[r.integers(0, len(letters), n)]) for n in lens]
    pick = np.minimum(r.zipf(1.3, words) - 1, vocab - 1)
    seps = [b" ", b"  ", b", ", b". ", b"\n", b" 42 ", b"\xc3\xa9"]
    out = []
    for i, w in enumerate(pick):
        out.append(voc[w])
        out.append(seps[int(r.integers(0, len(seps)))] if r.random() < 0.3 else b" ")
    return b"".join(out)


def tel_dict(t):
    return {"max_depth": t.max_depth, "nodes": t.nodes, "scratch_moves": t.scratch_moves,
            "bucket_assignments": t.bucket_assignments, "scratch_allocations": t.scratch_allocations,
            "matrix_cells_by_level": {str(k): v for k, v in sorted(t.matrix_cells_by_level.items())}}


def main():
    z: dict[str, np.ndarray] = {}
    meta: dict = {"texts": [], "sorts": [], "aggs": []}
    # 1. content-hash known answers
    r = np.random.default_rng(7)
    strings = [b"", b"a", b"the cat", b"\x00", b"\xff\xfe", bytes(range(256))]
    strings += [bytes(r.integers(0, 256, int(n), dtype=np.uint8)) for n in r.integers(0, 41, 120)]
    z["kat_blob"] = np.frombuffer(b"".join(strings), dtype=np.uint8)
    z["kat_len"] = np.array([len(s) for s in strings], dtype=np.uint64)
    z["kat_hash"] = np.array([hash_bytes(s) for s in strings], dtype=np.uint64)
    arena = r.integers(0, 256, 5000, dtype=np.uint8)
    offs = r.integers(0, 4900, 3000).astype(np.uint64)
    lens = r.integers(0, 100, 3000).astype(np.uint64)
    z["pre_arena"], z["pre_off"], z["pre_len"] = arena, offs, lens
    z["pre_hash"] = BytePrefixHasher(arena).hash_views(offs, lens)
    # 2. build_ngrams outputs
    texts = [("cats", b"The cat. the dog", 2), ("abab", b"a b a b a c a b", 2), ("four", b"one two three four", 3),
             ("nonascii", "Café au lait — déjà vu".encode(), 2), ("empty", b"", 2),
             ("digits", b"...123...", 2), ("synth", synth_text(3, 3000, 80), 3)]
    for name, text, g in texts:
        rec = build_ngrams(text, g)
        z[f"text_{name}"] = np.frombuffer(text, dtype=np.uint8)
        z[f"ng_{name}_arena"] = np.asarray(rec.arena, dtype=np.uint8)
        z[f"ng_{name}_keys"] = np.asarray(rec.keys, dtype=np.uint64).reshape(-1, 2)
        z[f"ng_{name}_values"] = np.asarray(rec.values, dtype=np.uint64).reshape(-1, 2)
        meta["texts"].append({"name": name, "gram": g})
    # 3. semisort of n-gram records
    corpora = [("small", synth_text(11, 20000, 300), 2, dict(light_buckets=16, base_case_cutoff=64, max_heavy=8)),
               ("tri", synth_text(12, 20000, 300), 3, dict(light_buckets=16, base_case_cutoff=64, max_heavy=8)),
               ("dflt", synth_text(13, 30000, 2000), 2, {})]
    for name, text, g, kw in corpora:
        z[f"corpus_{name}"] = np.frombuffer(text, dtype=np.uint8)
        rec = build_ngrams(text, g)
        n = len(rec)
        z[f"cng_{name}_arena"] = np.asarray(rec.arena, dtype=np.uint8)
        z[f"cng_{name}_keys"] = np.asarray(rec.keys, dtype=np.uint64).reshape(-1, 2)
        z[f"cng_{name}_values"] = np.asarray(rec.values, dtype=np.uint64).reshape(-1, 2)
        for mode in ("eq", "lt"):
            data = rec.copy()
            tel = S.Telemetry()
            S.semisort(data, ngram_adapter(rec), mode, S.TuningParams.for_input(n, **kw), telemetry=tel)
            z[f"sort_{name}_{mode}_keys"] = np.asarray(data.keys, dtype=np.uint64)
            z[f"sort_{name}_{mode}_values"] = np.asarray(data.values, dtype=np.uint64)
            meta["sorts"].append({"name": name, "gram": g, "mode": mode, "params": kw, "telemetry": tel_dict(tel)})
        # 4. aggregates (counts; wrapping sums of the value views' first word)
        for kind in ("count", "sum64"):
            tel = S.Telemetry()
            params = S.TuningParams.for_input(n, **kw)
            if kind == "count":
                res = S.histogram(rec, ngram_adapter(rec), params, telemetry=tel)
            else:
                res = S.collect_reduce(rec, ngram_adapter(rec), S.ReduceSpec.summing64(), params, telemetry=tel)
            pairs = sorted(res.pairs)
            meta["aggs"].append({"name": name, "gram": g, "kind": kind, "params": kw, "telemetry": tel_dict(tel),
                                 "pairs": [[k.decode("latin-1"), int(v)] for k, v in pairs]})
    z["meta"] = np.array(json.dumps(meta, sort_keys=True))
    np.savez_compressed(os.path.join(HERE, "golden_bytes.npz"), **z)
    print(len(meta["sorts"]), "sorts,", len(meta["aggs"]), "aggregates,", len(texts), "texts")


if __name__ == "__main__":
    main()
