#!/bin/bash
# Widened domain + large-match tests, then A/B of kMaxCompCams 32 (product) vs 16 (variant) at cfg3 and cfg1.
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider --timeout 900 2>&1 | tail -4
bash scripts/ab.sh
CFG=cfg1 STEPS=300 bash scripts/ab.sh
