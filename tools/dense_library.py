import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
import bench_suite
print(json.dumps(bench_suite.dense_library_record(), indent=1))
