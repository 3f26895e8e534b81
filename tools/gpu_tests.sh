# GPU test pass: the new / changed tests first (fail fast), then the whole -m gpu suite, smoke.
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "nonsymmetric or concurrent or stream_ordered or stress or config_full_size" 2>&1 | tail -15
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8
python __graft_entry__.py smoke 2>&1 | tail -2
