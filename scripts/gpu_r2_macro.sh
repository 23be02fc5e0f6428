#!/usr/bin/env bash
timeout 900 python -m pytest tests/test_gpu_macro.py -q 2>&1 | grep -v "^  " | tail -40
