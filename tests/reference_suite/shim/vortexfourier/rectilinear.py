from paper_1605_01244_b200.rectilinear import *  # noqa: F401,F403
