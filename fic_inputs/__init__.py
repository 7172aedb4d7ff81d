"""Seeded synthetic inputs and run configurations shared by the oracle and the CUDA path.

Holds no arithmetic of the method; see synth.py for the image recipe.
"""
from .synth import make_image, ramp_image, constant_image, random_image, sample_indices  # noqa: F401
from .configs import config, image_for, levels, s_sets, PREDEFINED_S, GRID_S, SAMPLED10_S, CLOSED5_S  # noqa: F401
