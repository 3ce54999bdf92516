python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cd oracle/_ref && timeout 1500 python -m pytest -p tests.refsuite_shim tests -q -x --co -q 2>&1 | tail -3; cd ../..
PYTHONPATH=$PWD timeout 1500 python -m pytest -p tests.refsuite_shim oracle/_ref/tests -q -rfE --junitxml=gpurun_out/refsuite.xml -o cache_dir=/tmp/pc > gpurun_out/refsuite.log 2>&1
tail -60 gpurun_out/refsuite.log
