# build ab/libttb_base.so from a git revision (default HEAD~1) for tools/ab.sh
rev=${1:-HEAD~1}
rm -rf /tmp/abpkg && mkdir -p /tmp/abpkg && git archive "$rev" paper_2507_14668_b200 include | tar -x -C /tmp/abpkg
(cd /tmp/abpkg && python -m paper_2507_14668_b200.build --force > /dev/null 2>&1)
mkdir -p ab && cp /tmp/abpkg/paper_2507_14668_b200/libttb.so ab/libttb_base.so && echo "ab/libttb_base.so <- $rev"
