#!/bin/bash
# build helper: fails loudly
cd /root/repo && python -m paper_2303_14102_b200.build > /tmp/build.log 2>&1 || { grep -E "error" -A3 /tmp/build.log | head -30; exit 1; }
echo built
