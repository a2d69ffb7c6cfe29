"""Print the bank-aware schedule quality for the config-1 network (host only)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
