"""Merge reference pins of the SURVEY §8(d) field H(n) into golden_hashes.json.

The pins come from the UNMODIFIED reference run on the GPU host (196 GB RAM,
16 cores): scripts/ref_pin.py (H(2^24), H(2^26), H(2^27) through
oracle/_ref's ref_dbscan) and scripts/ref_pin_big.py (H(2^30) through
oracle/_ref's ref_fof_field, all in one process).  Their raw JSON outputs are
committed under profiles/r02/; this script copies the hashes, counts and the
bench checksum into tests/golden/golden_hashes.json under "H_2^k".

    python tests/golden/pin_fields.py profiles/r02/ref_pin.json [profiles/r02/ref_pin_big.json]
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KEEP = ("n", "points_hash", "clusters", "noise", "core", "core_hash", "labels_hash", "labels_checksum",
        "ref_seconds", "threads")


def main():
    path = os.path.join(HERE, "golden_hashes.json")
    g = json.load(open(path))
    for src in sys.argv[1:]:
        for key, v in json.load(open(src)).items():
            entry = {k: v[k] for k in KEEP if k in v}
            entry["_source"] = "oracle/_ref friends_of_friends on H(%d), %s" % (v["n"], os.path.basename(src))
            g[key] = entry
    with open(path, "w") as f:
        json.dump(g, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
