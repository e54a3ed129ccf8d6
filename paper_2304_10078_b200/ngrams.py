"""N-gram records over cleaned text, built on the device (ngrams.py of the
reference).

Cleaning (ngrams.py:23-62): ASCII letters are lowercased and kept, every
other byte (digits, punctuation, non-ASCII) separates words; the words are
packed into an arena joined by single spaces.  A gram of g words is the
record (key = view of its first g-1 words, which are contiguous in the
arena; value = view of its last word) (ngrams.py:65-89).  Keys group by
content through BytesKeyAdapter (bytes_keys.py).  Everything after the text
upload runs as torch device ops; outputs equal the reference's arrays.
"""

from __future__ import annotations

import numpy as np
import torch

from .adapters import BytesKeyAdapter
from .errors import ConfigurationError
from .records import RecordArray, default_device

_SPACE = 0x20


def _text_tensor(text, device) -> torch.Tensor:
    if isinstance(text, str):
        text = text.encode("utf-8", errors="replace")
    raw = np.frombuffer(bytes(text), dtype=np.uint8)
    return torch.from_numpy(raw.copy()).to(device)


def clean_words(text, device=None):
    """(arena uint8, word offsets uint64, word lengths uint64), on the device."""
    dev = device or default_device()
    t = _text_tensor(text, dev).to(torch.int32)
    low = torch.where((t >= ord("A")) & (t <= ord("Z")), t + 32, t)
    alpha = (low >= ord("a")) & (low <= ord("z"))
    empty = torch.zeros(0, dtype=torch.uint64, device=dev)
    if t.numel() == 0 or not bool(alpha.any()):
        return torch.zeros(0, dtype=torch.uint8, device=dev), empty, empty
    prev = torch.cat([torch.zeros(1, dtype=torch.bool, device=dev), alpha[:-1]])
    nxt = torch.cat([alpha[1:], torch.zeros(1, dtype=torch.bool, device=dev)])
    src_start = torch.nonzero(alpha & ~prev).flatten()        # first letter of each word
    src_end = torch.nonzero(alpha & ~nxt).flatten() + 1        # one past its last letter
    length = src_end - src_start
    dst_start = torch.cumsum(length + 1, 0) - (length + 1)     # words joined by one space
    size = int((dst_start[-1] + length[-1]).item())
    arena = torch.full((size,), _SPACE, dtype=torch.uint8, device=dev)
    pos = torch.nonzero(alpha).flatten()                       # every letter, in text order
    word = torch.cumsum((alpha & ~prev).to(torch.int64), 0)[pos] - 1
    arena[dst_start[word] + (pos - src_start[word])] = low[pos].to(torch.uint8)
    return arena, dst_start.to(torch.int64).view(torch.uint64), length.to(torch.int64).view(torch.uint64)


def build_ngrams(text, gram_size: int, device=None) -> RecordArray:
    """One record per window of gram_size consecutive words (ngrams.py:65-89)."""
    if gram_size < 2:
        raise ConfigurationError("gram_size must be >= 2")
    arena, starts, lengths = clean_words(text, device)
    dev = arena.device
    s = starts.view(torch.int64)
    ln = lengths.view(torch.int64)
    count = max(0, int(s.numel()) - gram_size + 1)
    keys = torch.zeros((count, 2), dtype=torch.int64, device=dev)
    values = torch.zeros((count, 2), dtype=torch.int64, device=dev)
    if count:
        h = gram_size - 1
        keys[:, 0] = s[:count]
        keys[:, 1] = s[h - 1:h - 1 + count] + ln[h - 1:h - 1 + count] - s[:count]
        values[:, 0] = s[h:h + count]
        values[:, 1] = ln[h:h + count]
    return RecordArray(keys.view(torch.uint64), values.view(torch.uint64), "bytes", arena)


def ngram_adapter(records: RecordArray) -> BytesKeyAdapter:
    return BytesKeyAdapter(records.arena)


def decode_view(arena, view) -> str:
    buf = arena.cpu().numpy() if isinstance(arena, torch.Tensor) else np.asarray(arena, dtype=np.uint8)
    off, length = int(view[0]), int(view[1])
    return buf[off:off + length].tobytes().decode("latin-1")
