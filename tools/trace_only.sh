python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/trace_frame.py 40 C2 > gpurun_out/trace_x.txt 2>&1
python tools/trace_frame.py 150 C2 >> gpurun_out/trace_x.txt 2>&1
