"""Fixtures shared by several test modules (rotations of the reference's conftest.py:16-23)."""
import numpy as np

from paper_2205_07976_b200 import MosaicDomainSet


def rotation_about(axis, angle_deg):
    axis = np.asarray(axis, dtype=float)
    axis = axis / np.linalg.norm(axis)
    ang = np.radians(angle_deg)
    ax, ay, az = axis
    k = np.array([[0, -az, ay], [az, 0, -ax], [-ay, ax, 0]])
    return np.eye(3) + np.sin(ang) * k + (1 - np.cos(ang)) * (k @ k)


def two_domain_mosaic():
    return MosaicDomainSet(np.stack([rotation_about([1, 0, 0], 0.02), rotation_about([0, 1, 1], -0.03)]),
                           spread_deg=0.03)
