# SASS of one kernel of the library: tools/sass_fn.sh <mangled-name-substring> [lib]
lib=${2:-paper_1712_09005_b200/libfitsne_b200.so}
cuobjdump -sass "$lib" 2>/dev/null | awk -v pat="$1" '
  /Function :/ { on = index($0, pat) > 0 }
  on && /^\s+\/\*[0-9a-f]{4}\*\// { sub(/^\s+/, ""); sub(/\s*\/\* 0x[0-9a-f]* \*\/$/, ""); print }'
