#!/bin/sh
# Builds the CPU oracle (test infrastructure).  -ffp-contract=off and no
# -ffast-math are REQUIRED: the f32 canonical operation order
# must be evaluated one correctly-rounded op at a time.
set -e
cd "$(dirname "$0")"
g++ -O2 -std=c++17 -fopenmp -ffp-contract=off -fno-fast-math -fPIC -shared \
    -Wall -Wextra -o libgg_oracle.so gg_oracle.cpp
