#!/bin/bash
cd "$GRAFT_REPO_ROOT"
bash tools/r02_gpu_suite.sh ${1:-r02h}
bash tools/r02_profiles.sh ${2:-r02g}
