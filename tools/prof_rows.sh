timeout 300 ncu --set full --clock-control none --import-source on -k regex:sc_rows -s 3 -c 1 -o gpurun_out/prof_rows_five python tools/sc_case.py five > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sc_rows -s 3 -c 1 -o gpurun_out/prof_rows_syn python tools/sc_case.py synthetic > /dev/null 2>&1
