"""Time one secondary BASELINE config (dev helper): python tools/time_secondary.py c4"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import json
import sys

import bench

print(json.dumps(bench.time_secondary(sys.argv[1], steps=int(sys.argv[2]) if len(sys.argv) > 2 else 3)))
