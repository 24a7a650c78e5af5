"""f4: the artifact's on-disk formats and the host builders that feed them.

SURVEY.md §8f row 4. Three formats, all defined only by the reference's SPEC
(the reference's proj/ headers implement none of them):

  frequency table  SPEC.md:245  `gram<TAB>corpus_freq<TAB>doc_freq`, one row per
                   line, sorted corpus_freq desc then gram asc; '#' lines ignored.
                   Built on the GPU: corpus_freq and doc_freq are per-term
                   reductions over the count rows (refsig_gpu_get_corpus_freq,
                   refsig_gpu_get_df); only the 17,576-row sort is host work.
  MRCREF           SPEC.md:338  `MRCREF 1 <P> <L> <provenance>` then L grams;
                   partitions follow from the ceil rule.
  MRCS             SPEC.md:401  per-document signature file, written for every
                   document at once by the device (refsig_gpu_get_signature_records).

The reference builders (all / nonzero / band / infogain /
partition) are included because a Reference is what set_reference_vectors()
consumes; they are O(17,576) host work on a table, not on documents.

Gap decisions (DESIGN.md §1 f4):
  * MRCS header: the field list (4 + 4 + 4 + 8) is 20 bytes; SPEC.md:401's
    closing sentence says "24 bytes total", which no listed field accounts for.
    The field list is normative here: header 20 bytes, payload at offset 20.
  * partition(): SPEC requires every partition non-empty and the first P-1 of
    size ceil(L/P); when (P-1)*ceil(L/P) >= L (e.g. L=9, P=4) both cannot hold
    and partition() raises ValidationError instead of emitting an empty one.
  * ref_id = FNV-1a 64 of the canonical MRCREF bytes, i.e. what
    save_reference() writes (LF line ends), so a loaded reference and the one
    that was saved have the same id.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field

import numpy as np

from . import ValidationError

GRAM_LEN = 3
GRAM_SPACE = 26 ** 3
MRCS_MAGIC = b"MRCS"
MRCS_VERSION = 1
MRCS_HEADER = 20
MRCREF_MAGIC = "MRCREF"
MRCREF_VERSION = 1

_FNV_OFFSET = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3
_MASK64 = (1 << 64) - 1


# -- grams ---------------------------------------------------------------------
def is_gram(s: str) -> bool:
    """ngram.hpp:25-30: exactly three 'a'..'z'."""
    return len(s) == GRAM_LEN and all("a" <= c <= "z" for c in s)


def pack_gram(s: str) -> int:
    """ngram.hpp:32-36: base-26 id, so id order == lexicographic order."""
    if not is_gram(s):
        raise ValidationError(f'not a 3-gram: "{s}"')
    return ((ord(s[0]) - 97) * 26 + (ord(s[1]) - 97)) * 26 + (ord(s[2]) - 97)


def unpack_gram(i: int) -> str:
    """ngram.hpp:38-45."""
    i = int(i)
    if not 0 <= i < GRAM_SPACE:
        raise ValidationError(f"gram id {i} outside [0, {GRAM_SPACE})")
    return chr(97 + i // 676) + chr(97 + (i // 26) % 26) + chr(97 + i % 26)


def fnv1a64(data: bytes) -> int:
    """FNV-1a 64 (offset basis 0xcbf29ce484222325, prime 0x100000001b3)."""
    h = _FNV_OFFSET
    for b in data:
        h = ((h ^ b) * _FNV_PRIME) & _MASK64
    return h


# -- frequency table ---------------------------------------------
@dataclass(eq=False)
class FrequencyTable:
    """Rows (gram id, corpus_freq, doc_freq), sorted cf desc then gram asc."""
    gram: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    cf: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    df: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))

    def __len__(self) -> int:
        return len(self.gram)

    def __eq__(self, o) -> bool:
        return (isinstance(o, FrequencyTable) and np.array_equal(self.gram, o.gram)
                and np.array_equal(self.cf, o.cf) and np.array_equal(self.df, o.df))

    def rows(self) -> list[tuple[str, int, int]]:
        return [(unpack_gram(g), int(c), int(d)) for g, c, d in zip(self.gram, self.cf, self.df)]

    @staticmethod
    def from_rows(rows) -> "FrequencyTable":
        """From (gram str, cf, df) tuples in any order; validates and sorts."""
        g = np.array([pack_gram(r[0]) for r in rows], np.uint32)
        cf = np.array([int(r[1]) for r in rows], np.uint64)
        df = np.array([int(r[2]) for r in rows], np.uint64)
        if len(np.unique(g)) != len(g):
            raise ValidationError("duplicate gram in frequency rows")
        if np.any(df < 1) or np.any(cf < df):
            raise ValidationError("frequency rows need corpus_freq >= doc_freq >= 1")
        return FrequencyTable._sorted(g, cf, df)

    @staticmethod
    def from_counts(cf: np.ndarray, df: np.ndarray) -> "FrequencyTable":
        """From dense per-gram-id cf/df vectors (length 17,576); keeps cf > 0."""
        cf = np.asarray(cf, np.uint64)
        df = np.asarray(df, np.uint64)
        if len(cf) != GRAM_SPACE or len(df) != GRAM_SPACE:
            raise ValidationError(f"frequency vectors must have {GRAM_SPACE} entries (3-gram vocabulary)")
        g = np.flatnonzero(cf).astype(np.uint32)
        if np.any(df[g] < 1) or np.any(cf[g] < df[g]) or np.any(df[cf == 0] != 0):
            raise ValidationError("inconsistent corpus_freq / doc_freq vectors")
        return FrequencyTable._sorted(g, cf[g], df[g])

    @staticmethod
    def _sorted(g, cf, df) -> "FrequencyTable":
        o = np.lexsort((g, np.iinfo(np.uint64).max - cf))  # cf desc, then gram asc
        return FrequencyTable(np.ascontiguousarray(g[o]), np.ascontiguousarray(cf[o]), np.ascontiguousarray(df[o]))


def build_frequency_table(ctx) -> FrequencyTable:
    """build_frequency_table for the corpus loaded in ctx
    (load_text()/load_corpus() with the 3-gram vocabulary, then count())."""
    if getattr(ctx, "vocab", None) != GRAM_SPACE:
        raise ValidationError(f"frequency tables are over the 3-gram vocabulary ({GRAM_SPACE} terms)")
    cf = ctx.corpus_freq()
    df, _ = ctx.df()
    return FrequencyTable.from_counts(cf, df.astype(np.uint64))


def dumps_frequency_table(t: FrequencyTable) -> str:
    return "".join(f"{unpack_gram(g)}\t{int(c)}\t{int(d)}\n" for g, c, d in zip(t.gram, t.cf, t.df))


def loads_frequency_table(text: str) -> FrequencyTable:
    """Parse SPEC.md:245; every error names its 1-based line."""
    g, cf, df = [], [], []
    seen = set()
    for n, line in enumerate(text.splitlines(), 1):
        if line.startswith("#"):
            continue
        f = line.split("\t")
        if len(f) != 3:
            raise ValidationError(f"wrong field count ({len(f)}, expected 3) at line {n}")
        if len(f[0]) != GRAM_LEN:
            raise ValidationError(f"gram length ≠ 3 at line {n}")
        if not is_gram(f[0]):
            raise ValidationError(f'gram "{f[0]}" is not 3 lowercase letters at line {n}')
        if not (f[1].isascii() and f[1].isdigit() and f[2].isascii() and f[2].isdigit()):
            raise ValidationError(f"non-integer frequency at line {n}")
        gi, c, d = pack_gram(f[0]), int(f[1]), int(f[2])
        if c >= 1 << 64 or d >= 1 << 64:
            raise ValidationError(f"frequency exceeds 64 bits at line {n}")
        if d < 1 or c < d:
            raise ValidationError(f"need corpus_freq >= doc_freq >= 1 at line {n}")
        if gi in seen:
            raise ValidationError(f"duplicate gram at line {n}")
        if g and (c > cf[-1] or (c == cf[-1] and gi < g[-1])):
            raise ValidationError(f"rows not sorted (corpus_freq desc, gram asc) at line {n}")
        seen.add(gi)
        g.append(gi)
        cf.append(c)
        df.append(d)
    return FrequencyTable(np.array(g, np.uint32), np.array(cf, np.uint64), np.array(df, np.uint64))


def save_frequency_table(t: FrequencyTable, path) -> None:
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write(dumps_frequency_table(t))


def load_frequency_table(path) -> FrequencyTable:
    with open(path, encoding="utf-8") as fh:
        return loads_frequency_table(fh.read())


# -- gram lists and references ---------------------------------
@dataclass(eq=False)
class GramList:
    grams: np.ndarray
    provenance: str

    def __len__(self) -> int:
        return len(self.grams)

    def __eq__(self, o) -> bool:
        return isinstance(o, GramList) and self.provenance == o.provenance and np.array_equal(self.grams, o.grams)


def build_all() -> GramList:
    """all 17,576 grams, lexicographic."""
    return GramList(np.arange(GRAM_SPACE, dtype=np.uint32), "all")


def build_nonzero(t: FrequencyTable) -> GramList:
    """the table's grams in its descending-frequency order."""
    if len(t) == 0:
        raise ValidationError("empty frequency table")
    return GramList(t.gram.copy(), "nonzero")


def build_band(t: FrequencyTable, lo: int, hi: int) -> GramList:
    """slice [lo, hi) of the nonzero list."""
    if not 0 <= lo < hi:
        raise ValidationError(f"band needs 0 <= lo < hi (got {lo}, {hi})")
    if hi > len(t):
        raise ValidationError(f"band hi={hi} exceeds the nonzero list length {len(t)}")
    return GramList(t.gram[lo:hi].copy(), f"band({lo},{hi})")


def build_infogain(t: FrequencyTable, k: int) -> GramList:
    """rank by (doc_freq asc, corpus_freq asc, gram asc), take k."""
    if k < 1:
        raise ValidationError("infogain needs k >= 1")
    if k > len(t):
        raise ValidationError(f"infogain k={k} exceeds the {len(t)} grams available")
    o = np.lexsort((t.gram, t.cf, t.df))
    return GramList(np.ascontiguousarray(t.gram[o[:k]]), f"infogain({k})")


def partition_sizes(L: int, p: int) -> list[int]:
    """Ceil rule: P-1 chunks of ceil(L/P), then the rest."""
    if p < 1 or p > L:
        raise ValidationError(f"partition count {p} outside [1, {L}]")
    c = -(-L // p)
    last = L - c * (p - 1)
    if last < 1:
        raise ValidationError(f"ceil rule leaves the last partition empty (L={L}, P={p}, chunk {c})")
    return [c] * (p - 1) + [last]


@dataclass(eq=False)
class Reference:
    """Gram list + P contiguous ceil-rule partitions (count 1 per gram)."""
    grams: GramList
    P: int

    def __post_init__(self):
        g = np.asarray(self.grams.grams)
        if len(np.unique(g)) != len(g):
            raise ValidationError("reference grams must be distinct")
        if len(g) and int(g.max()) >= GRAM_SPACE:
            raise ValidationError("reference gram id outside the 3-gram space")
        self.sizes = partition_sizes(len(g), self.P)

    def __eq__(self, o) -> bool:
        return isinstance(o, Reference) and self.P == o.P and self.grams == o.grams

    @property
    def L(self) -> int:
        return len(self.grams)

    @property
    def rowptr(self) -> np.ndarray:
        r = np.zeros(self.P + 1, np.uint64)
        r[1:] = np.cumsum(self.sizes)
        return r

    @property
    def partitions(self) -> list[np.ndarray]:
        r = self.rowptr
        return [self.grams.grams[int(r[i]):int(r[i + 1])] for i in range(self.P)]

    def canonical_bytes(self) -> bytes:
        return dumps_reference(self).encode("ascii")

    @property
    def ref_id(self) -> int:
        return fnv1a64(self.canonical_bytes())

    def install(self, ctx) -> None:
        """Upload the partition vectors (count 1 per gram) as the K = P references."""
        ctx.set_reference_vectors(self.rowptr, np.asarray(self.grams.grams, np.uint32), None)


def partition(grams: GramList, p: int) -> Reference:
    return Reference(grams, int(p))


def dumps_reference(ref: Reference) -> str:
    prov = ref.grams.provenance
    if not prov or any(c.isspace() for c in prov):
        raise ValidationError("provenance must be one non-empty token")
    head = f"{MRCREF_MAGIC} {MRCREF_VERSION} {ref.P} {ref.L} {prov}\n"
    return head + "".join(unpack_gram(g) + "\n" for g in ref.grams.grams)


def loads_reference(text: str) -> Reference:
    lines = text.splitlines()
    if not lines:
        raise ValidationError("empty reference file")
    h = lines[0].split(" ")
    if h[0] != MRCREF_MAGIC:
        raise ValidationError(f"bad magic (expected {MRCREF_MAGIC}) at line 1")
    if len(h) != 5:
        raise ValidationError(f"header needs 5 fields, got {len(h)} at line 1")
    if h[1] != str(MRCREF_VERSION):
        raise ValidationError(f"unsupported MRCREF version {h[1]!r} at line 1")
    if not (h[2].isascii() and h[2].isdigit() and h[3].isascii() and h[3].isdigit()):
        raise ValidationError("non-integer P or L at line 1")
    P, L = int(h[2]), int(h[3])
    if P < 1:
        raise ValidationError(f"P={P} must be >= 1 at line 1")
    if len(lines) - 1 != L:
        raise ValidationError(f"gram-count mismatch: header L={L}, file has {len(lines) - 1} grams")
    g = np.empty(L, np.uint32)
    seen = set()
    for n in range(2, L + 2):
        s = lines[n - 1]
        if not is_gram(s):
            raise ValidationError(f'not a 3-gram "{s}" at line {n}')
        gi = pack_gram(s)
        if gi in seen:
            raise ValidationError(f"duplicate gram at line {n}")
        seen.add(gi)
        g[n - 2] = gi
    return Reference(GramList(g, h[4]), P)


def save_reference(ref: Reference, path) -> None:
    with open(path, "wb") as fh:
        fh.write(ref.canonical_bytes())


def load_reference(path) -> Reference:
    with open(path, "rb") as fh:
        data = fh.read()
    try:
        text = data.decode("utf-8")
    except UnicodeDecodeError as e:
        raise ValidationError(f"reference file is not UTF-8: {e}") from None
    return loads_reference(text)


# -- MRCS signature files --------------------------------------------
def _mrcs_dtype(P: int) -> np.dtype:
    return np.dtype([("magic", "S4"), ("version", "<u4"), ("P", "<u4"), ("ref_id", "<u8"), ("v", "<f8", (P,))])


def encode_signature(values, ref_id: int) -> bytes:
    v = np.ascontiguousarray(values, "<f8").ravel()
    return MRCS_MAGIC + struct.pack("<IIQ", MRCS_VERSION, len(v), int(ref_id) & _MASK64) + v.tobytes()


def decode_signature(data: bytes) -> tuple[np.ndarray, int]:
    """-> (float64 values, ref_id)."""
    if len(data) < MRCS_HEADER or data[:4] != MRCS_MAGIC:
        raise ValidationError("bad magic (expected MRCS)")
    ver, P, ref_id = struct.unpack_from("<IIQ", data, 4)
    if ver != MRCS_VERSION:
        raise ValidationError(f"unsupported MRCS version {ver}")
    if len(data) != MRCS_HEADER + 8 * P:
        raise ValidationError(f"MRCS size {len(data)} != {MRCS_HEADER} + 8*P (P={P})")
    return np.frombuffer(data, "<f8", P, MRCS_HEADER).copy(), ref_id


def decode_records(rec: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """uint8 [N, 20 + 8P] (Context.signature_records) -> (f64 [N, P], ref_id [N])."""
    rec = np.ascontiguousarray(rec, np.uint8)
    if rec.ndim != 2 or rec.shape[1] < MRCS_HEADER or (rec.shape[1] - MRCS_HEADER) % 8:
        raise ValidationError("records must be uint8 [N, 20 + 8P]")
    P = (rec.shape[1] - MRCS_HEADER) // 8
    r = rec.view(_mrcs_dtype(P)).reshape(len(rec))
    if np.any(r["magic"] != MRCS_MAGIC) or np.any(r["version"] != MRCS_VERSION) or np.any(r["P"] != P):
        raise ValidationError("malformed MRCS record header")
    return np.ascontiguousarray(r["v"]), np.ascontiguousarray(r["ref_id"])


def check_same_reference(ref_id_a: int, ref_id_b: int) -> None:
    """compare()'s precondition: both signed on one reference."""
    if int(ref_id_a) != int(ref_id_b):
        raise ValidationError(f"signature ref_id mismatch ({int(ref_id_a):#018x} vs {int(ref_id_b):#018x})")


def save_signature(path, values, ref_id: int) -> None:
    with open(path, "wb") as fh:
        fh.write(encode_signature(values, ref_id))


def load_signature(path) -> tuple[np.ndarray, int]:
    with open(path, "rb") as fh:
        return decode_signature(fh.read())


def write_signature_files(directory, names, rec: np.ndarray) -> None:
    """One MRCS file per document from device-written records."""
    os.makedirs(directory, exist_ok=True)
    rec = np.ascontiguousarray(rec, np.uint8)
    if len(names) != len(rec):
        raise ValidationError("one name per record")
    for n, r in zip(names, rec):
        with open(os.path.join(directory, n), "wb") as fh:
            fh.write(r.tobytes())
