python tests/gpu_microbench.py 2>&1 | grep -E "^(nt_|post_|dcomp|update|neg)" | cut -c1-100
