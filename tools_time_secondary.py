"""Time one secondary BASELINE config (dev helper): python tools_time_secondary.py c4"""
import json
import sys

import bench

print(json.dumps(bench.time_secondary(sys.argv[1], steps=int(sys.argv[2]) if len(sys.argv) > 2 else 3)))
