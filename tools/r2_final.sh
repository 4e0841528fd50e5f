#!/bin/bash
# Round-2 final evidence on one B200: tools/r2_round.sh (tests, smoke, bench lines, launch list,
# traffic, ncu K1a / K1b) followed by tools/r2_gpu_b.sh (host packing, C3 shard, 2 / 4 ranks, sanitizer).
tools/r2_round.sh ${1:-r2k}
tools/r2_gpu_b.sh ${1:-r2k}b
