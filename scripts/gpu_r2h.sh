#!/bin/bash
# Drop-in StitchEngine + details-in-flight: unit/acceptance suites, engine bench, rig tests.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_engine_dropin.py tests/test_reference_unit_tests.py tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "engine or reference or in_flight or cfg1 or graph or failed or cache" 2>&1 | tail -25
