"""Builders for the hand-derived scenarios in tests/golden/scenarios.json."""
import json
import os

import numpy as np

import tracegen as tg

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scenarios.json")
ATTN_ONLY = tg.Model(4, 0, 4)
MODELS = {"7B": tg.MODEL_7B, "attn_only": ATTN_ONLY}


def load():
    with open(GOLDEN) as f:
        return json.load(f)


def _blocks(spec):
    names = sorted(spec["blocks"])
    return {nm: [10_000 * (i + 1) + j for j in range(spec["blocks"][nm])] for i, nm in enumerate(names)}


def _expand(items, blocks):
    out = []
    for it in items:
        if it.startswith("#"):
            out.append(int(it[1:]))
        elif ":" in it:
            nm, k = it.split(":")
            out.extend(blocks[nm][:int(k)])
        else:
            out.extend(blocks[it])
    return out


def scenario_trace(spec, sc):
    b = _blocks(spec)
    reqs = [(_expand(i, b), _expand(o, b)) for i, o in sc["requests"]]
    return tg.from_sequences(reqs, name=sc["name"])


def variant(sc):
    cap = sc.get("cap_bytes")
    return tg.Variant(MODELS[sc["model"]], tg.UNLIMITED_BYTES if cap is None else cap, sc.get("cap_nodes", 0))


def eviction_example(spec, ex):
    """(trace, snapshot nodes structured array fields, next_id) for E1/E2."""
    b = _blocks(spec)
    reqs = [(_expand(s, b), []) for s in ex["seqs"]]
    tr = tg.from_sequences(reqs, name=ex["name"])
    nodes = []
    for (nid, par, si, ds, de, t, ssm) in ex["snapshot"]:
        nodes.append((nid, par, int(tr.off[si]), ds, de, t, ssm))
    return tr, nodes, ex["next_id"]
