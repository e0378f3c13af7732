python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python tools/build_variants.py dbg=-DDEBUG_SYNC > /dev/null
echo "=== dbg"; SCALESIM_SO=$PWD/build/variants/dbg.so timeout 300 python tools/big_debug.py 2>&1 | tail -14
