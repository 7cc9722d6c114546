#!/bin/sh
# Registers / stack / static shared memory per kernel of a libinim.so build (default: in-tree).
LIB=${1:-$(dirname "$0")/../paper_2408_06513_b200/libinim.so}
/usr/local/cuda/bin/cuobjdump -res-usage "$LIB" 2>/dev/null | awk '
  /Function/ { name = $2; sub(":$", "", name); next }
  /REG:/ && name != "" { print $1, $2, $3, name; name = "" }' | c++filt | sed 's/(.*//' | sort -k4
