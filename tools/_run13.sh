NK_LIB_PATH=paper_2103_16400_b200/libnttkit_b200_tl.so timeout 300 python tools/timeline_str.py
NK_LIB_PATH=paper_2103_16400_b200/libnttkit_b200_tl.so timeout 300 python tools/timeline_stri.py
