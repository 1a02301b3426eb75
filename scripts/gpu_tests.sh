set -o pipefail
timeout 1200 python -m pytest tests -m gpu -x -q -k "${1:-}" 2>&1 | tail -40
