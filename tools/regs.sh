#!/bin/bash
# registers / smem per kernel of an object or .so: tools/regs.sh <file> [pattern]
cuobjdump -res-usage "$1" 2>/dev/null | awk '/Function/ {name=$2} /REG:/ {print $0, name}' | grep -E "${2:-.}" | sed -E 's/STACK:0 //; s/TEXTURE:0 SURFACE:0 SAMPLER:0//' | c++filt | cut -c1-200
