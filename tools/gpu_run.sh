#!/bin/bash
# dev helper: rebuild the extension, then run a command on the GPU box
cd /root/repo || exit 1
if python paper_2203_15561_b200/build.py 2>&1 | grep -iE "error|errno"; then exit 1; fi
timeout 2400 /usr/local/graft/bin/gpurun --timeout "${T:-900}" -- "$@" 2>&1 | grep -v "^\[gpurun\] send"
