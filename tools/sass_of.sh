#!/bin/bash
# usage: tools/sass_of.sh lib.so 'ILi7ELi8ELb0E' out.sass  — SASS of one k_sweep_v2 instance
cuobjdump -sass "$1" | awk -v pat="k_sweep_v2$2" '/Function :/ {on = index($0, pat) > 0} on' > "$3"
cuobjdump -res-usage "$1" 2>/dev/null | grep -A1 "k_sweep_v2$2" | tail -1
