# usage: bash tools/sass_count.sh <lib.so>   static SASS opcode histogram of fast_step_kernel<1,4,false>
fn=$(cuobjdump -symbols "$1" | grep -oE "_ZN3scb[A-Za-z0-9_]*fast_step_kernelILb1ELi4ELb0EEE[A-Za-z0-9_]*" | head -1)
cuobjdump -sass -fun "$fn" "$1" 2>/dev/null | grep -oE "^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[0-9T] )?[A-Z0-9.]+" | awk '{print $NF}' | sed 's/\..*//' | sort | uniq -c | sort -rn | head -${2:-16}
