"""CSV files of the command-line pipelines, same formats as the reference
(datapipe.py:392-470): numeric feature matrices with an optional header line,
single-column 1-based class IDs (0 = unlabeled), `node_id,class_id`
predictions, %.17g score / value matrices."""

import csv

import numpy as np

from .errors import FormatError


def _rows(path):
    try:
        with open(path, newline="", encoding="utf-8") as fh:
            rows = list(csv.reader(fh))
    except csv.Error as exc:
        raise FormatError(f"{path}: malformed CSV ({exc})") from exc
    return [r for r in rows if r and any(c.strip() for c in r)]


def _has_header(first, parse):
    try:
        for cell in first:
            parse(cell)
        return False
    except ValueError:
        return True


def load_features_csv(path):
    """(n, D) float64; a non-numeric first line is a header."""
    rows = _rows(path)
    if not rows:
        raise FormatError(f"{path}: empty feature file")
    skip = 1 if _has_header(rows[0], float) else 0
    body = rows[skip:]
    if not body:
        raise FormatError(f"{path}: header line but no data rows")
    width = len(body[0])
    out = np.empty((len(body), width))
    for i, row in enumerate(body):
        line = i + skip + 1
        if len(row) != width:
            raise FormatError(f"{path}:{line}: expected {width} columns, found {len(row)}")
        try:
            out[i] = [float(c) for c in row]
        except ValueError as exc:
            raise FormatError(f"{path}:{line}: non-numeric value ({exc})") from exc
    return out


def load_labels_csv(path, n=None):
    """0-based class IDs, -1 where the file says 0 (unlabeled)."""
    rows = _rows(path)
    if not rows:
        raise FormatError(f"{path}: empty label file")
    skip = 1 if _has_header(rows[0][:1], int) else 0
    body = rows[skip:]
    ids = np.empty(len(body), dtype=np.int64)
    for i, row in enumerate(body):
        line = i + skip + 1
        if len(row) != 1:
            raise FormatError(f"{path}:{line}: expected a single column, found {len(row)}")
        try:
            c = int(row[0])
        except ValueError as exc:
            raise FormatError(f"{path}:{line}: non-integer class ID ({exc})") from exc
        if c < 0:
            raise FormatError(f"{path}:{line}: class IDs are 1-based with 0 = unlabeled, got {c}")
        ids[i] = c - 1
    if n is not None and ids.shape[0] != n:
        raise FormatError(f"{path}: {ids.shape[0]} labels for {n} nodes")
    return ids


def write_predictions_csv(path, predictions):
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("node_id,class_id\n")
        fh.writelines(f"{i},{int(c) + 1}\n" for i, c in enumerate(np.asarray(predictions)))


def write_matrix_csv(path, values):
    np.savetxt(path, np.asarray(values), fmt="%.17g", delimiter=",")
