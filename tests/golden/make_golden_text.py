"""Golden vectors for the text layer from the UNMODIFIED reference ``tinfer.bench``
(build container only; ``/root/reference`` is absent on the GPU box).

    python tests/golden/make_golden_text.py   # -> tests/golden/text.json

The reference ships no ``tinfer/tokenizer.py``, so its ``bench.py``
is loaded with this repo's tokenizer registered as ``tinfer_ref.tokenizer``;
``gen_vocab`` / ``gen_dataset`` / ``sample_lengths`` / ``choose_keep_count``
only use the ``Vocab`` container from it, so the recorded words, texts and
lengths are the reference's own SplitMix64-driven output.
"""

from __future__ import annotations

import importlib.util
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref_loader  # noqa: E402
from paper_2407_04991_b200 import tokenizer as our_tok  # noqa: E402

T = ref_loader.load()
sys.modules["tinfer_ref.tokenizer"] = our_tok
T.tokenizer = our_tok
for n in ("pruning", "pipeline", "graphopt", "bench"):
    spec = importlib.util.spec_from_file_location(f"tinfer_ref.{n}", f"{ref_loader.REF_SRC}/{n}.py")
    m = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = m
    spec.loader.exec_module(m)
    setattr(T, n, m)
B = T.bench


def main():
    out = {}
    v = B.gen_vocab(128, seed=9)
    out["vocab_128_9"] = list(v.tokens)
    out["vocab_4096_42_head"] = list(B.gen_vocab(4096, seed=42).tokens[:64])
    out["dataset_40_4_12_30"] = B.gen_dataset(40, seed=4, mean=12, max_len=30, vocab=v)
    out["lengths_2000_123"] = B.sample_lengths(2000, T.rng.SplitMix64(123), mean=60, max_len=100)
    v256 = B.gen_vocab(256, seed=3)
    texts = B.gen_dataset(40, seed=5, mean=20, max_len=60, vocab=v256)
    counts = T.pruning.scan_frequencies(texts, our_tok.build(v256))
    out["keep_count_256_3"] = int(B.choose_keep_count(counts, 0.99, sorted(v256.special_ids)))
    with open(os.path.join(HERE, "text.json"), "w", encoding="utf-8") as fh:
        json.dump(out, fh, ensure_ascii=False, sort_keys=True)
    print("wrote text.json")


if __name__ == "__main__":
    main()
