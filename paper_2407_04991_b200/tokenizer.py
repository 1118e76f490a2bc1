"""Greedy longest-match trie tokenizer (the paper's Faster-Tokenizer stand-in).

The reference package imports ``tinfer.tokenizer`` (pipeline.py:28,
pruning.py:21, bench.py:59) but does not ship it; its API and behaviour are
restated from the reference's own tests and spec:

* ``Vocab(tokens, unk, eos, pad, frequency=None)`` — frozen, comparable;
  ``VocabError`` for an empty or duplicate token, equal specials, or a special
  outside ``[0, len)`` (test_tokenizer.py:35-50);
* ``build(vocab) -> Tokenizer`` — a code-point trie;
* ``Tokenizer.encode`` — left-to-right greedy longest match, no match emits
  ``unk`` and advances one code point, whitespace is an ordinary character
  (test_tokenizer.py:53-79);
* ``Tokenizer.decode`` — concatenation, ``unk`` renders as U+FFFD, an id out of
  range raises ``VocabError`` (test_tokenizer.py:82-98);
* ``read_vocab`` / ``write_vocab`` — UTF-8 TSV with a ``#unk=/#eos=/#pad=``
  header, then ``token<TAB>frequency`` per line, id = line index; byte-exact
  round trip; ``FormatError`` on a missing header, a tab or newline inside a
  token, or a bad frequency (test_tokenizer.py:120-154).

Host-side by design: tokenisation happens once per request before the batch is
formed and is not on the GPU hot path.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Sequence

from .errors import FormatError, VocabError

UNK_RENDER = "�"
_END = ""  # trie key marking a terminal node (tokens are never empty)


@dataclass(frozen=True)
class Vocab:
    tokens: tuple[str, ...]
    unk: int
    eos: int
    pad: int
    frequency: tuple[int, ...] | None = None

    def __post_init__(self):
        object.__setattr__(self, "tokens", tuple(self.tokens))
        if self.frequency is not None:
            object.__setattr__(self, "frequency", tuple(int(f) for f in self.frequency))
            if len(self.frequency) != len(self.tokens):
                raise VocabError("frequency must have one entry per token")
        n = len(self.tokens)
        seen: set[str] = set()
        for t in self.tokens:
            if not isinstance(t, str) or not t:
                raise VocabError("tokens must be non-empty strings")
            if t in seen:
                raise VocabError(f"duplicate token {t!r}")
            seen.add(t)
        for name in ("unk", "eos", "pad"):
            sid = getattr(self, name)
            if not isinstance(sid, int) or not 0 <= sid < n:
                raise VocabError(f"{name} id {sid!r} out of range [0, {n})")
        if len({self.unk, self.eos, self.pad}) != 3:
            raise VocabError("unk, eos and pad must be distinct ids")

    def __len__(self) -> int:
        return len(self.tokens)

    @property
    def special_ids(self) -> set[int]:
        return {self.unk, self.eos, self.pad}


class Tokenizer:
    """Immutable after :func:`build`; safe to share across threads."""

    def __init__(self, vocab: Vocab):
        self.vocab = vocab
        root: dict = {}
        for tid, tok in enumerate(vocab.tokens):
            node = root
            for ch in tok:
                node = node.setdefault(ch, {})
            node[_END] = tid
        self._root = root
        self._tokens = vocab.tokens

    def encode(self, text: str) -> list[int]:
        root, unk = self._root, self.vocab.unk
        out: list[int] = []
        i, n = 0, len(text)
        while i < n:
            node = root
            best_id, best_end = unk, i + 1
            j = i
            while j < n:
                node = node.get(text[j])
                if node is None:
                    break
                j += 1
                tid = node.get(_END)
                if tid is not None:
                    best_id, best_end = tid, j
            out.append(best_id)
            i = best_end
        return out

    def decode(self, ids: Iterable[int]) -> str:
        toks, n, unk = self._tokens, len(self._tokens), self.vocab.unk
        parts = []
        for i in ids:
            i = int(i)
            if not 0 <= i < n:
                raise VocabError(f"token id {i} out of range [0, {n})")
            parts.append(UNK_RENDER if i == unk else toks[i])
        return "".join(parts)


def build(vocab: Vocab) -> Tokenizer:
    return Tokenizer(vocab)


def write_vocab(path: str | Path, vocab: Vocab) -> None:
    lines = [f"#unk={vocab.unk}", f"#eos={vocab.eos}", f"#pad={vocab.pad}"]
    freq: Sequence[int] = vocab.frequency if vocab.frequency is not None else (0,) * len(vocab)
    for tok, f in zip(vocab.tokens, freq):
        if "\t" in tok or "\n" in tok or "\r" in tok:
            raise FormatError(f"token {tok!r} contains a tab or line break")
        lines.append(f"{tok}\t{int(f)}")
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


def read_vocab(path: str | Path) -> Vocab:
    with open(path, "r", encoding="utf-8", newline="\n") as fh:
        lines = fh.read().split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    specials = {}
    for k, name in enumerate(("unk", "eos", "pad")):
        if k >= len(lines) or not lines[k].startswith(f"#{name}="):
            raise FormatError(f"vocab header line {k}: expected '#{name}=<id>'")
        try:
            specials[name] = int(lines[k][len(name) + 2:])
        except ValueError:
            raise FormatError(f"vocab header line {k}: bad id") from None
    tokens, freq = [], []
    for ln, line in enumerate(lines[3:], start=3):
        tok, sep, f = line.rpartition("\t")
        if not sep:
            raise FormatError(f"vocab line {ln}: expected token<TAB>frequency")
        if "\t" in tok:
            raise FormatError(f"vocab line {ln}: tab inside a token")
        try:
            fv = int(f)
        except ValueError:
            raise FormatError(f"vocab line {ln}: bad frequency {f!r}") from None
        if fv < 0 or str(fv) != f:
            raise FormatError(f"vocab line {ln}: bad frequency {f!r}")
        tokens.append(tok)
        freq.append(fv)
    return Vocab(tokens=tuple(tokens), unk=specials["unk"], eos=specials["eos"],
                 pad=specials["pad"], frequency=tuple(freq))
