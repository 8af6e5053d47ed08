#!/usr/bin/env python
"""Small-problem latency: bench.py's cfg1 us/call and SP2 on cfg1-sized H (device and host loops)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2102_08505_b200 as eb  # noqa: E402

eb.build()
print(json.dumps(bench.time_cfg1(eb, 0, 300)))
print(json.dumps(bench.time_sp2_small(eb, 0, 20, "cfg1")))
print(json.dumps(bench.time_sp2_small(eb, 0, 20, "soft_matter")))
