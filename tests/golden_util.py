"""Loaders for the committed golden fixtures (made by oracle/gen_golden.py)."""
import functools
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(None)
def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def engine_cases():
    return load("engine_cases.json")["cases"]


def case_by_name(name):
    for c in engine_cases():
        if c["name"] == name:
            return c
    raise KeyError(name)
