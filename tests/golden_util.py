"""Loading helpers for tests/golden (fixtures produced by tools/make_golden.py from the
reference ftlz package)."""

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def sha(buf) -> str:
    return hashlib.sha256(memoryview(np.ascontiguousarray(buf)).cast("B")).hexdigest()


def faults_of(entry):
    return [tuple(f) for f in entry.get("faults", [])]


def override_of(entry):
    ov = entry.get("override") or {}
    return {int(k): int(v) for k, v in ov.items()} or None
