#!/bin/bash
# per-phase build_amg device times (CF_TIMING=1) for the config-3 u-hierarchy
CF_TIMING=1 python scripts/amg_ab.py cfg3 2>&1 | grep "^\[amg" | tail -60
