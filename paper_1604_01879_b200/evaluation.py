"""Retrieval metrics of `evaluate_index` (reference evaluation.py:44-88):
nearest neighbour, first and second tier, mean average precision and the
area under the 11-point interpolated precision-recall curve.  Computed from
the 1-based ranks of a query's relevant shapes (the query itself excluded),
which the GPU ranking produces directly."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import NoValidQueries, SingletonClass

RECALL_LEVELS = np.linspace(0.0, 1.0, 11)
AUC_DEFINITION = "trapezoid under the 11-point interpolated mean precision-recall curve"


@dataclass(frozen=True)
class QueryMetrics:
    nn: float
    ft: float
    st: float
    ap: float
    pr11: np.ndarray


@dataclass(frozen=True)
class EvalReport:
    nn: float
    ft: float
    st: float
    map: float
    auc: float
    pr11: np.ndarray
    n_queries: int
    n_skipped: int = 0


def metrics_from_ranks(ranks, class_size: int, label: str = "") -> QueryMetrics:
    """`ranks`: ascending 1-based positions of the relevant shapes in the
    query's ranking (query excluded); `class_size` counts the query."""
    n_rel = class_size - 1
    if n_rel < 1:
        raise SingletonClass(f"class of {label!r} has no other member")
    ranks = np.asarray(ranks, dtype=np.int64)
    nn = 1.0 if len(ranks) and ranks[0] == 1 else 0.0
    ft = float(np.count_nonzero(ranks <= n_rel)) / n_rel
    st = float(np.count_nonzero(ranks <= 2 * n_rel)) / n_rel
    hits = np.arange(1, len(ranks) + 1)
    prec = hits / ranks if len(ranks) else np.zeros(0)
    ap = float(prec.sum()) / n_rel
    rec = hits / n_rel
    pr11 = np.array([float(prec[rec >= lv - 1e-12].max()) if np.any(rec >= lv - 1e-12) else 0.0
                     for lv in RECALL_LEVELS])
    return QueryMetrics(nn=nn, ft=ft, st=st, ap=ap, pr11=pr11)


def score_ranking(query_label: str, ranked_labels, class_size: int) -> QueryMetrics:
    """Reference signature (evaluation.py:44): ranked labels of one query."""
    rel = np.flatnonzero(np.array([lab == query_label for lab in ranked_labels], dtype=bool))
    return metrics_from_ranks(rel + 1, class_size, query_label)


def aggregate_report(per_query, n_skipped: int = 0) -> EvalReport:
    per_query = list(per_query)
    if not per_query:
        raise NoValidQueries("no valid queries to aggregate")
    pr11 = np.mean([m.pr11 for m in per_query], axis=0)
    return EvalReport(nn=float(np.mean([m.nn for m in per_query])),
                      ft=float(np.mean([m.ft for m in per_query])),
                      st=float(np.mean([m.st for m in per_query])),
                      map=float(np.mean([m.ap for m in per_query])),
                      auc=float(np.trapezoid(pr11, RECALL_LEVELS)), pr11=pr11,
                      n_queries=len(per_query), n_skipped=n_skipped)


def report_to_dict(report: EvalReport, extra: dict | None = None) -> dict:
    out = {"auc_definition": AUC_DEFINITION, "n_queries": report.n_queries,
           "n_skipped": report.n_skipped, "NN": report.nn, "FT": report.ft, "ST": report.st,
           "MAP": report.map, "AUC": report.auc,
           "pr_recall": [float(r) for r in RECALL_LEVELS],
           "pr_precision": [float(p) for p in report.pr11]}
    if extra:
        out.update(extra)
    return out
