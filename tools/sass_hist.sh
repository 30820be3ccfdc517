#!/bin/bash
# static SASS opcode histogram of the kernels matching $2 in object/library $1
obj=$1; pat=$2
cuobjdump -sass "$obj" | awk -v pat="$pat" '/Function :/{on = ($0 ~ pat)} on' \
  | grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9_.]+" | awk '{print $NF}' | sed 's/\..*//' \
  | sort | uniq -c | sort -rn
