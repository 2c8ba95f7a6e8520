#!/bin/bash
# usage: tools/sass_loop.sh <obj> <function-regex> <anchor-mnemonic> [before] [after]
# Prints the instruction histogram of the SASS window around the first anchor.
cd "$(dirname "$0")/.."
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{f=($0 ~ pat)} f' | sed 's|/\* 0x[0-9a-f]* \*/||;s|^\s*/\*[0-9a-f]*\*/||' | grep -v "^\s*$" > /tmp/_fn.sass
L=$(grep -n "$3" /tmp/_fn.sass | head -1 | cut -d: -f1)
B=${4:-20}; A=${5:-80}
awk -v s=$((L-B)) -v e=$((L+A)) 'NR>=s && NR<=e' /tmp/_fn.sass > /tmp/_win.sass
awk '{print $1}' /tmp/_win.sass | sed 's/^@.*//' | sort | uniq -c | sort -rn | head -14
