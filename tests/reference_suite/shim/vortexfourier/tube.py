from paper_1605_01244_b200.tube import *  # noqa: F401,F403
