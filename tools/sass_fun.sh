#!/bin/bash
# usage: tools/sass_fun.sh <binary> <function-substring>  -> SASS of the first matching function
cuobjdump -sass "$1" | awk -v pat="$2" '/Function :/ {p = index($0, pat) > 0} p'
