"""Record sha256 digests of the reference's DIMACS fixture files with the
generate(...) parameters that pin them (reference test_io_cli.py:154-164), so the
package's own generator + serializer can be checked byte-for-byte without the
reference present.  Run here: python tests/golden/make_fixture_hashes.py"""

import hashlib
import json
import os

FIX = "/root/reference/pkg/tests/fixtures"
SPECS = {
    "maxflow_small.max": ["maxflow", 12, 25, 50, 7],
    "maxflow_medium.max": ["maxflow", 60, 250, 100, 11],
    "maxflow_fixed.max": ["maxflow", 40, 160, 100, 77],
    "assign_complete_n5.asn": ["assignment", 5, None, 100, 3],
    "assign_sparse_n6.asn": ["assignment", 6, 0.5, 100, 9],
    "assign_fixed_n8.asn": ["assignment", 8, None, 100, 77],
}
out = {}
for name, spec in SPECS.items():
    text = open(os.path.join(FIX, name), encoding="utf-8").read()
    out[name] = {"generate": spec, "sha256": hashlib.sha256(text.encode()).hexdigest(), "bytes": len(text)}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "fixture_hashes.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1)[:400])
