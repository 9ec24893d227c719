# usage: fsass.sh lib.so pattern -> SASS of the first function whose name matches
cuobjdump -sass $1 2>/dev/null | awk -v pat="$2" '/Function :/{p = ($3 ~ pat) && !done; if(p) done=1} p' | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed 's@/\* 0x[0-9a-f]* \*/@@'
