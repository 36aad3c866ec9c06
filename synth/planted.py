"""synth.planted -- seeded planted-topic corpus with journal labels (NEXT-4).

INPUT GENERATION ONLY (no step of the method's arithmetic).  Stands in for the
PubMed journal corpus of P:247-249 (five BMC journals, 20,112 terms, 7,510
abstracts after stop-word removal), which is not available: each document
belongs to one of ``n_journals`` journals (balanced, shuffled) and draws
``tokens`` term occurrences, each with probability ``mix`` from its journal's
topic distribution (a Zipf law over a journal-specific random subset of
``topic_terms`` terms) and otherwise from a shared background Zipf law over the
``common`` fraction of the vocabulary (the generic words that row normalisation
is meant to de-emphasise); the topic subsets are drawn from the rest and
may overlap.  Entries are occurrence counts a_ij ("the number of
times term i occurs in document j"); terms that occur only once in the corpus
are dropped, their rows left empty.  Row normalisation is NOT
applied here: it is a step of the method (esnmf_options.row_normalize,
oracle.normalize_rows).
"""
from __future__ import annotations

import numpy as np


def _zipf_cdf(n: int, s: float) -> np.ndarray:
    w = 1.0 / np.arange(1, n + 1, dtype=np.float64) ** s
    c = np.cumsum(w)
    return c / c[-1]


def _csr(rows: np.ndarray, cols: np.ndarray, vals: np.ndarray, nrows: int):
    order = np.lexsort((cols, rows))
    r, c, v = rows[order], cols[order], vals[order]
    ptr = np.zeros(nrows + 1, np.int64)
    np.add.at(ptr, r + 1, 1)
    return np.cumsum(ptr), c.astype(np.int32), v.astype(np.float32)


def planted_corpus(n_terms: int = 20_112, n_docs: int = 7_510, n_journals: int = 5, tokens: int = 120,
                   topic_terms: int = 4_000, mix: float = 0.5, common: float = 0.1, s: float = 1.05,
                   seed: int = 0) -> dict:
    """Returns dict(n, m, a_ptr, a_col, a_val, at_ptr, at_col, at_val, labels, n_journals)."""
    rng = np.random.default_rng(seed)
    labels = rng.permutation(np.arange(n_docs) % n_journals).astype(np.int32)
    n_common = max(1, int(common * n_terms))
    bg_cdf = _zipf_cdf(n_common, s)
    tp_cdf = _zipf_cdf(topic_terms, s)
    topic = np.stack([n_common + rng.choice(n_terms - n_common, topic_terms, replace=False)
                      for _ in range(n_journals)])
    from_topic = rng.random((n_docs, tokens)) < mix
    bg = np.minimum(np.searchsorted(bg_cdf, rng.random((n_docs, tokens))), n_common - 1)
    tr = np.minimum(np.searchsorted(tp_cdf, rng.random((n_docs, tokens))), topic_terms - 1)
    term = np.where(from_topic, topic[labels[:, None], tr], bg)
    doc = np.repeat(np.arange(n_docs), tokens)
    key, cnt = np.unique(doc.astype(np.int64) * n_terms + term.ravel(), return_counts=True)
    d, t = key // n_terms, key % n_terms
    # drop terms occurring only once in the whole corpus
    occ = np.bincount(t, weights=cnt, minlength=n_terms)
    keep = occ[t] > 1
    d, t, cnt = d[keep], t[keep], cnt[keep]
    a_ptr, a_col, a_val = _csr(t, d, cnt, n_terms)
    at_ptr, at_col, at_val = _csr(d, t, cnt, n_docs)
    return dict(n=n_terms, m=n_docs, a_ptr=a_ptr, a_col=a_col, a_val=a_val, at_ptr=at_ptr, at_col=at_col,
                at_val=at_val, labels=labels, n_journals=n_journals)
