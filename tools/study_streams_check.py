"""Prints the ErrorStats of two multi-chunk studies (chunks of 2^20): run under KOG2_STUDY_STREAMS=0/1/2 the output must not change."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_13116_b200 import capi, configs
from paper_2407_13116_b200 import kogsvd2 as K
capi.load().kog_study_set_chunk_log2(20)
for c in (configs.cfg(5, count=5 * (1 << 20) + 77), configs.cfg(4, count=2 * (1 << 20) + 5)):
    s = K.StudyStats(); s.add(c, 0, c.count); print(bytes(s.read()).hex()[:64], K.csv_row(c, s.read())[-60:])
