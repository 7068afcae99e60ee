#!/bin/bash
# The reference acceptance suite's LORBPANO_CLI_PATH for the B200 build: the
# lorbpano command line of this repo (paper_1810_03988_b200/cli.py).
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
cd "$ROOT" 2>/dev/null && exec python -m paper_1810_03988_b200 "$@"
