from .planner import *
