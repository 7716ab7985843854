#!/bin/bash
# Static SASS instruction count of one function in an object/library.
# Usage: tools/sass_count.sh OBJ MANGLED_NAME
cuobjdump -sass "$1" 2>/dev/null | awk -v f="$2" '/Function :/{p=($3==f)} p && /^ +\/\*[0-9a-f]+\*\/ /{c++} END{print c+0}'
