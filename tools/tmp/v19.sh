timeout 600 python tools/gen_mesh_bench.py 32 48 2>&1 | cut -c1-420
timeout 900 python -m pytest tests -m gpu -x -q -k "mesh" 2>&1 | tail -3
