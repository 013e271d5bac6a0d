ACI_LIB=tools/libab/libaci_ts.so timeout 200 python tools/time_chi.py 256 2 2>&1 | grep -E "ts b=|chi=" | tail -45
ACI_LIB=tools/libab/libaci_ts.so timeout 200 python tools/time_chi.py 64 2 2>&1 | grep -E "ts b=|chi=" | tail -45
