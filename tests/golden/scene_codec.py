"""Encode narrow-phase inputs/outputs for fixtures; decode into the
package's duck-typed body classes (the GPU box has no reference)."""

from __future__ import annotations

import numpy as np

from paper_2309_15417_b200 import bodies as B


def encode_tree(tree, dedup=False):
    """Levels as arrays.  With `dedup`, the fine level's corners are stored
    as unique vertices plus int32 corner indices (the fine corners are the
    mesh's recentred vertices gathered per face, so this is lossless) and a
    constant epsilon as one value: large meshes stay small on disk."""
    levels = []
    for li, lvl in enumerate(tree.levels):
        corners = np.asarray(lvl.corners, dtype=np.float64)
        eps = np.asarray(lvl.epsilon, dtype=np.float64)
        if dedup and li == 0:
            v, inv = np.unique(corners.reshape(-1, 3), axis=0, return_inverse=True)
            rec = {"fine_v": v, "fine_f": inv.reshape(-1, 3).astype(np.int32)}
            assert np.array_equal(v[rec["fine_f"]].view(np.uint64), corners.view(np.uint64))
            if len(eps) and np.all(eps.view(np.uint64) == eps[:1].view(np.uint64)):
                rec["epsilon_const"] = float(eps[0])
            else:
                rec["epsilon"] = eps
        else:
            rec = {"corners": corners, "epsilon": eps}
        if lvl.children is not None:
            ch = [np.asarray(c, dtype=np.int64) for c in lvl.children]
            rec["child_ptr"] = np.cumsum([0] + [len(c) for c in ch]).astype(np.int64)
            rec["child_idx"] = np.concatenate(ch) if ch else np.zeros(0, np.int64)
        levels.append(rec)
    return levels


def decode_tree(levels):
    out = []
    for rec in levels:
        children = None
        if "child_ptr" in rec:
            ptr, idx = rec["child_ptr"], rec["child_idx"]
            children = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
        if "fine_v" in rec:
            corners = np.ascontiguousarray(rec["fine_v"][rec["fine_f"]])
            eps = rec["epsilon"] if "epsilon" in rec else np.full(len(corners), rec["epsilon_const"])
        else:
            corners, eps = rec["corners"], rec["epsilon"]
        out.append(B.SurrogateLevel(corners=np.asarray(corners), epsilon=np.asarray(eps), children=children))
    return B.SurrogateTree(levels=out)


def encode_body(body, dedup=False):
    if hasattr(body, "timeline"):
        s = body.timeline.current
        return {"kind": "particle", "id": int(body.pid), "tree": encode_tree(body.tree, dedup),
                "epsilon": float(body.epsilon),
                "position": np.asarray(s.position, float), "velocity": np.asarray(s.velocity, float),
                "rotation": np.asarray(s.rotation, float),
                "angular_velocity": np.asarray(s.angular_velocity, float), "t": float(s.t)}
    return {"kind": "static", "id": int(body.sid), "tree": encode_tree(body.tree, dedup),
            "epsilon": float(body.epsilon)}


def decode_body(rec):
    tree = decode_tree(rec["tree"])
    if rec["kind"] == "particle":
        st = B.state(rec["position"], rec["velocity"], rec["rotation"], rec["angular_velocity"],
                     rec["t"])
        return B.Particle(pid=rec["id"], tree=tree, epsilon=rec["epsilon"], radius=0.0,
                          timeline=B.timeline(st))
    return B.StaticBody(sid=rec["id"], tree=tree, epsilon=rec["epsilon"])


CONTACT_FIELDS = ("body_a", "body_b", "position", "normal", "depth", "t", "tri_a", "tri_b",
                  "threshold")


def encode_contacts(contacts):
    n = len(contacts)
    return {
        "body_a": np.array([c.body_a for c in contacts], dtype=np.int64),
        "body_b": np.array([c.body_b for c in contacts], dtype=np.int64),
        "position": np.array([np.asarray(c.position, float) for c in contacts]).reshape(n, 3),
        "normal": np.array([np.asarray(c.normal, float) for c in contacts]).reshape(n, 3),
        "depth": np.array([c.depth for c in contacts], dtype=np.float64),
        "t": np.array([c.t for c in contacts], dtype=np.float64),
        "tri_a": np.array([c.tri_a for c in contacts], dtype=np.int64),
        "tri_b": np.array([c.tri_b for c in contacts], dtype=np.int64),
        "threshold": np.array([c.threshold for c in contacts], dtype=np.float64),
    }


def encode_result(res, raw):
    return {"dt": float(res.dt), "collision": bool(res.collision),
            "first_contact": None if res.first_contact is None else float(res.first_contact),
            "narrowing_iters": int(res.narrowing_iters),
            "bound_history": np.array(res.bound_history, dtype=np.float64),
            "contacts": encode_contacts(res.contacts), "raw": encode_contacts(raw)}
