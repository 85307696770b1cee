timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "cpp_host or nvcc" 2>&1 | tail -5
